"""Host time per call of sf_filter on cfg1 (256^2), back to back, measured on
the host clock: the Python binding (validation + ctypes) against the bare
ctypes call into libsf.so, and the GPU-side time per call of the same loop
(events).  Prints one JSON object."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1107_4617_b200 as sf  # noqa: E402
import synth  # noqa: E402
from bench import _image  # noqa: E402

dev = torch.device("cuda:0")
c = synth.CONFIGS["cfg1"]
img = torch.from_numpy(_image(c)).to(dev)
o = torch.empty((c.H, c.W), dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
lib = sf.load()
import ctypes  # noqa: E402

h = ctypes.c_void_p(st.cuda_stream)


def wrapped():
    sf.sf_filter(img, c.radius, c.kind, c.sigma_r, c.N, out=o, stream=st)


def bare():
    lib.sf_filter(ctypes.c_void_p(img.data_ptr()), c.H, c.W, c.radius, c.kind, c.sigma_r, c.N,
                  ctypes.c_void_p(o.data_ptr()), h)


res = {}
for name, fn in (("binding", wrapped), ("bare_ctypes", bare)):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    res[name] = {"host_us_per_call": (t1 - t0) / n * 1e6, "gpu_us_per_call": e0.elapsed_time(e1) / n * 1e3}
print(json.dumps(res))
