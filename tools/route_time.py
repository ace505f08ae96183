"""Router kernel timing: lane-per-token vs four-lanes-per-token (Qwen3 shape)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200 import _lib
from paper_2508_09591_b200.layer import route_topk
lg = torch.randn(32768, 128, device="cuda")
for quad in (0, 1, 0, 1):
    _lib.call("hm_route_set_option", quad)
    for _ in range(5): route_topk(lg, 8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): route_topk(lg, 8)
    e1.record(); e1.synchronize()
    print(json.dumps({"quad": quad, "us": e0.elapsed_time(e1) / 50 * 1e3}))
