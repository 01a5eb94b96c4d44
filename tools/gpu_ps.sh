#!/bin/bash
# pair split (cluster of ps CTAs per unit, DSMEM reduction): parity on small
# images for ps = 1..4 and the cfg1 / cfg2 times
mkdir -p gpurun_out; O=gpurun_out/ps.log; : > $O
cat > /tmp/pspar.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1107_4617_b200 as sf, synth, oracle
worst = 0.0
for (H, W, N, s, seed) in [(256, 256, 30, 30.0, 5), (150, 530, 30, 30.0, 77), (40, 700, 66, 20.0, 3), (17, 1000, 118, 15.0, 9), (333, 517, 264, 10.0, 4), (130, 200, 264, 10.0, 4)]:
    img = synth.gen_image(H, W, seed, 10.0)
    t = torch.from_numpy(img).cuda()
    for r in (1, 2, 5, 8, 13, 16, 24):
        if r >= min(H, W): continue
        out = sf.sf_filter(t, r, 0, s, N).cpu().numpy().astype(np.float64)
        ref = oracle.bilateral_shiftable(img, r, 0, s, N)
        e = np.abs(out - ref)
        worst = max(worst, float(e.max()))
        print(H, W, N, "r", r, "max", float(e.max()), "mean", float(e.mean()), flush=True)
print("worst", worst)
PY
for ps in 1 2 3 4; do echo "-- parity ps=$ps" >> $O; SF_V7_PS=$ps timeout 300 python /tmp/pspar.py >> $O 2>&1; done
echo "-- parity auto" >> $O; timeout 300 python /tmp/pspar.py >> $O 2>&1
for ps in 1 2 3 4 auto; do
  echo "-- time ps=$ps" >> $O
  if [ $ps = auto ]; then timeout 300 python tools/time_cfg.py cfg1 5 cfg2 8 cfg3 10 >> $O 2>&1
  else SF_V7_PS=$ps timeout 300 python tools/time_cfg.py cfg1 5 cfg2 8 cfg3 10 >> $O 2>&1; fi
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_precision.py -x -q > gpurun_out/ps_tests.log 2>&1
tail -3 gpurun_out/ps_tests.log >> $O
