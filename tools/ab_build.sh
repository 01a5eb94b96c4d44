#!/bin/bash
# Build libsf.so of a git revision (default HEAD) into tools/_ab/libsf_<name>.so,
# for same-box A/B timing: SF_LIB_OVERRIDE=tools/_ab/libsf_base.so python tools/time_cfg.py ...
# (timings differ by up to ~10% between GPU boxes, so A/B runs belong in one call)
set -e
cd "$(dirname "$0")/.."
rev=${1:-HEAD}; name=${2:-base}
tmp=$(mktemp -d)
git archive "$rev" paper_1107_4617_b200/csrc include | tar -x -C "$tmp"
mkdir -p tools/_ab
python - "$tmp" "tools/_ab/libsf_$name.so" <<'PY'
import sys
from paper_1107_4617_b200 import _build
tmp, out = sys.argv[1], sys.argv[2]
_build.build(force=True, csrc=tmp + "/paper_1107_4617_b200/csrc", lib=out, objdir=tmp + "/objs")
PY
rm -rf "$tmp"
echo "tools/_ab/libsf_$name.so"
