"""The dispatch + combine step captured in a CUDA graph and replayed: the
barrier epochs live on the device, so replays keep working and give the
same bits as eager steps (all transports, one GPU)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dedup", ["gpu", "remote", "all", "none"])
def test_step_graph_replay(hm, dedup):
    from paper_2508_09591_b200.layer import EPWorld, route_topk
    G, E, K, M, T_r = 8, 64, 4, 512, 128
    ep = EPWorld(G, E, K, M, T_r)
    g = torch.Generator(device="cuda").manual_seed(3)
    xs = [torch.randn(G * T_r, M, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3)]
    ls = [torch.randn(G * T_r, E, device="cuda", generator=g) for _ in range(3)]
    x_in, l_in = xs[0].clone(), ls[0].clone()
    out = torch.empty_like(x_in)

    def step():
        slot, w, _ = route_topk(l_in, K)
        ep.dispatch(x_in, slot, w, dedup=dedup)
        ep.combine(slot, w, dedup=dedup, out=out)

    eager = []
    for x, lg in zip(xs, ls):
        x_in.copy_(x)
        l_in.copy_(lg)
        step()
        eager.append(out.clone())
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()                      # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(2):
        for x, lg, want in zip(xs, ls, eager):
            x_in.copy_(x)
            l_in.copy_(lg)
            graph.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, want)
    ep.check_status()
    ep.close()
