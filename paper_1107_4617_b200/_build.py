"""Build libsf.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Translation units: sf.cu (ABI, planner, the v1/v2/v4/v4r/q2/NLM tile
kernels), runtime.cu, v5_part.cu eight times (-DSF_V5_PART=0..7, the v5
kernel for radii 8i+1..8i+8), v7_part.cu and v7q_part.cu six times each (the
v7 box and v7q separable-q_M kernels for radii 4i+1..4i+4), v7w_part.cu eight
times (the wide large-radius v7 kernel for radii 25+5i..29+5i) and nlm_part.cu three times (-DSF_NLM_P=1..3,
the NLM band sweep); they are compiled in parallel to objects under build/
and linked into one shared library."""
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsf.so")
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, "sf.cu")]   # the ABI TU (tools compile it alone for ptxas reports)


def units(csrc: str):
    return [("sf", os.path.join(csrc, "sf.cu"), []), ("runtime", os.path.join(csrc, "runtime.cu"), [])] + \
        [(f"v5_part{i}", os.path.join(csrc, "v5_part.cu"), [f"-DSF_V5_PART={i}"]) for i in range(8)] + \
        [(f"v7_part{i}", os.path.join(csrc, "v7_part.cu"), [f"-DSF_V7_PART={i}"]) for i in range(6)] + \
        [(f"v7q_part{i}", os.path.join(csrc, "v7q_part.cu"), [f"-DSF_V7Q_PART={i}"]) for i in range(6)] + \
        [(f"v7w_part{i}", os.path.join(csrc, "v7w_part.cu"), [f"-DSF_V7W_PART={i}"]) for i in range(8)] + \
        [(f"nlm_part{i}", os.path.join(csrc, "nlm_part.cu"), [f"-DSF_NLM_P={i}"]) for i in (1, 2, 3)]


UNITS = units(CSRC)
OBJDIR = os.path.join(ROOT, "build", "objs")
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + \
    [os.path.join(ROOT, "include", "sf.h")]

COMPILE_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                 "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
NVCC_FLAGS = COMPILE_FLAGS + ["-shared"]   # single-TU compile (tools/spills.sh)


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _closure(src: str) -> set:
    """src and every file it #includes with quotes, transitively."""
    import re
    seen, todo = set(), [os.path.abspath(src)]
    while todo:
        f = todo.pop()
        if f in seen or not os.path.exists(f):
            continue
        seen.add(f)
        for inc in re.findall(r'^\s*#\s*include\s+"([^"]+)"', open(f).read(), re.M):
            todo.append(os.path.abspath(os.path.join(os.path.dirname(f), inc)))
    return seen


def build(force: bool = False, verbose: bool = False, csrc: str = None, lib: str = None, objdir: str = None) -> str:
    """Build the in-tree libsf.so (default), or — tools/ab_build.sh — another
    source tree `csrc` into `lib` with objects under `objdir`."""
    LIB_ = lib or LIB
    OBJDIR_ = objdir or OBJDIR
    UNITS_ = units(csrc) if csrc else UNITS
    stale = force or not os.path.exists(LIB_) or any(
        os.path.getmtime(d) > os.path.getmtime(LIB_) for d in DEPS if os.path.exists(d))
    if stale:
        os.makedirs(OBJDIR_, exist_ok=True)

        def compile_unit(u):
            name, src, defs = u
            obj = os.path.join(OBJDIR_, name + ".o")
            if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                    os.path.getmtime(d) for d in _closure(src)):
                return obj, ""                      # up to date (its own include closure)
            res = subprocess.run([nvcc()] + COMPILE_FLAGS + defs + ["-c", "-o", obj, src],
                                 capture_output=True, text=True)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed on {name}:\n" + res.stdout + res.stderr)
            return obj, res.stderr

        workers = max(1, min(len(UNITS_), os.cpu_count() or 1))
        with ThreadPoolExecutor(workers) as ex:
            done = list(ex.map(compile_unit, UNITS_))
        res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_] +
                             [o for o, _ in done], capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
        if verbose:
            for _, log in done:
                print(log)
    return LIB_


if __name__ == "__main__":
    print(build(force=True, verbose=True))
