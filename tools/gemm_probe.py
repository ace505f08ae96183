import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_2508_09591_b200 import _lib
from paper_2508_09591_b200.ffn import expert_ffn_ptrs, grouped_gemm
G, M, I = 16, 2048, 768
n = torch.full((G,), 2048, dtype=torch.int32, device="cuda")
rows = 32768; cap = rows + 256
x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
w13 = (torch.randn(G, 2*I, M, device="cuda") * M**-0.5).to(torch.bfloat16)
w2 = (torch.randn(G, M, I, device="cuda") * I**-0.5).to(torch.bfloat16)
h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / n
for stages in (6,):
  for skip in (0,):
    g1 = t(lambda: _lib.call("hm_grouped_gemm", x.data_ptr(), cap, w13.data_ptr(), G, n.data_ptr(), 2*I, M, 1, h.data_ptr(), I, _lib.stream_ptr()))
    g2 = t(lambda: _lib.call("hm_grouped_gemm", h.data_ptr(), cap, w2.data_ptr(), G, n.data_ptr(), M, I, 0, y.data_ptr(), M, _lib.stream_ptr()))
    print(json.dumps({"stages": stages, "skip_store": skip, "gemm1_ms": round(g1, 4), "gemm1_tf": round(2*rows*2*I*M/g1/1e9, 1), "gemm2_ms": round(g2, 4), "gemm2_tf": round(2*rows*M*I/g2/1e9, 1)}))
