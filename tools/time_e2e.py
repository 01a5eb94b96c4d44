"""End-to-end time of sf_filter_host (pinned host in/out, copies inside) on
cfg5 r=16: wall clock of 5 calls after one warm-up, as bench.py's e2e."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1107_4617_b200 as sf
import synth
c = synth.CONFIGS["cfg5"]
r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
h_in = torch.from_numpy(c.image()).pin_memory()
h_out = torch.empty(h_in.shape, dtype=torch.float32).pin_memory()
stream = torch.cuda.current_stream()
sf.sf_filter_host(h_in.numpy(), r, c.kind, c.sigma_r, c.N, out=h_out.numpy(), stream=stream)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    sf.sf_filter_host(h_in.numpy(), r, c.kind, c.sigma_r, c.N, out=h_out.numpy(), stream=stream)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"e2e_ms": round(sorted(ts)[2], 3), "all": [round(t, 3) for t in ts],
                  "lib": os.environ.get("SF_LIB_OVERRIDE", "in-tree")}))
