"""ptxas register/spill summary of the band-sweep kernels, per translation unit
(check before any GPU timing: spills inside the pair loop cost 10-30%).
usage: python tools/spills.py [filter]"""
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1107_4617_b200 import _build  # noqa: E402

flt = sys.argv[1] if len(sys.argv) > 1 else "box_v5"


def run(u):
    name, src, defs = u
    r = subprocess.run([_build.nvcc()] + _build.COMPILE_FLAGS + defs + ["-c", "-o", f"/tmp/_sp_{name}.o", src],
                       capture_output=True, text=True)
    return r.stderr.splitlines()


with ThreadPoolExecutor(8) as ex:
    logs = list(ex.map(run, _build.UNITS))
for lines in logs:
    for i, l in enumerate(lines):
        if "Compiling entry function" in l and flt in l:
            m = re.search(r"_ZN2sf\d+(\w+?)ILi(\d+)E(?:Lb(\d))?", l)
            name = f"{m.group(1)}<{m.group(2)}{',' + m.group(3) if m.group(3) else ''}>" if m else l
            sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", lines[i + 2])
            rg = re.search(r"Used (\d+) registers", lines[i + 3])
            print(f"{name:28s} regs {rg.group(1) if rg else '?':>4s}  spill st/ld {sp.group(1)}/{sp.group(2)}")
