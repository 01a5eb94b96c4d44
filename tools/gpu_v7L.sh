#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/v7L.log; : > $O
cat > /tmp/v7Lpar.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1107_4617_b200 as sf, synth, oracle
H, W, N, s, seed = 150, 530, 30, 30.0, 77
img = synth.gen_image(H, W, seed, 10.0)
t = torch.from_numpy(img).cuda()
worst = 0
for r in [25, 31, 32, 33, 40, 47, 56, 63, 64]:
    out = sf.sf_filter(t, r, 0, s, N).cpu().numpy().astype(np.float64)
    ref = oracle.bilateral_shiftable(img, r, 0, s, N)
    e = np.abs(out - ref)
    print("r", r, "max", float(e.max()), "mean", float(e.mean()), flush=True)
PY
echo "-- parity v7m large" >> $O; SF_VARIANT=v7m timeout 300 python /tmp/v7Lpar.py >> $O 2>&1
for v in v7m v5; do
  echo "-- $v" >> $O
  SF_VARIANT=$v timeout 300 python tools/time_cfg.py cfg5 64 cfg5 48 cfg5 32 cfg5 25 cfg5 16 cfg5 4 >> $O 2>&1
done
