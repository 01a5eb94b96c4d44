#!/bin/bash
# v7 bring-up: parity of v7 / v7m on small images, A/B timing against v5 / v6
mkdir -p gpurun_out; O=gpurun_out/v8.log; : > $O
cat > /tmp/v7par.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1107_4617_b200 as sf, synth, oracle
H, W, N, s, seed = 150, 530, 30, 30.0, 77
img = synth.gen_image(H, W, seed, 10.0)
t = torch.from_numpy(img).cuda()
for r in list(range(1, 25)):
    out = sf.sf_filter(t, r, 0, s, N).cpu().numpy().astype(np.float64)
    ref = oracle.bilateral_shiftable(img, r, 0, s, N)
    e = np.abs(out - ref)
    print("r", r, "max", float(e.max()), "mean", float(e.mean()), flush=True)
PY
for v in v8 v8m; do echo "-- parity $v" >> $O; SF_VARIANT=$v timeout 300 python /tmp/v7par.py >> $O 2>&1; done
for v in v7 v8 v8m; do
  echo "-- $v" >> $O
  SF_VARIANT=$v timeout 300 python tools/time_cfg.py cfg5 16 cfg5 4 cfg5 8 cfg4 16 >> $O 2>&1
done
echo "-- drift v8" >> $O
SF_VARIANT=v8 timeout 600 python tools/drift_stress.py >> $O 2>&1
