"""N = 1 dispatch+combine step (bench.py's headline, no layer / planner / CPU
arms) for A/B library builds: prints ms/step and the gather kernel time.
    HM_LIB=... python tools/gather_ab.py"""
import json
import subprocess
import sys

out = subprocess.run([sys.executable, "bench.py", "--steps", "100", "--warmup", "5", "--no-layer",
                      "--no-planner", "--no-cpu-baseline", "--no-e2e"], capture_output=True,
                     text=True)
line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
d = json.loads(line)
print(json.dumps({"ms_per_step": round(d["ms_per_step"], 4), "gather_ms": d["kernel_ms"]["gather"],
                  "graph_ms": d.get("cuda_graph_ms_per_step"), "roofline": d["roofline"]["frac"]}))
