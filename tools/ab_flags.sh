#!/bin/bash
# Build the working tree's libsf.so with extra nvcc flags into tools/_ab/libsf_<name>.so
# (same-box A/B of a compile-time option: SF_LIB_OVERRIDE=tools/_ab/libsf_<name>.so ...)
# usage: tools/ab_flags.sh NAME -DFOO=1 [...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/_ab
python - "$name" "$@" <<'PY'
import sys
from paper_1107_4617_b200 import _build
name, flags = sys.argv[1], sys.argv[2:]
_build.COMPILE_FLAGS = _build.COMPILE_FLAGS + flags
_build.build(force=True, lib=f"tools/_ab/libsf_{name}.so", objdir=f"build/ab_{name}")
PY
echo "tools/_ab/libsf_$name.so"
