#!/bin/bash
# usage: tools/sass_hist.sh <lib.so> <function-name-substring>
# Instruction histogram of one kernel's SASS (opcode without modifiers).
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/ {on = index($0, pat) > 0} on' \
  | grep -E "^\s+/\*[0-9a-f]+\*/" | sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+//; s/^@!?U?P[0-9T] //' \
  | awk '{print $1}' | sed 's/\..*//; s/;//' | sort | uniq -c | sort -rn
