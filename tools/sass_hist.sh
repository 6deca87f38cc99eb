#!/bin/bash
# Opcode histogram of one kernel's SASS in libgact.so: tools/sass_hist.sh <mangled-name-regex>
cuobjdump -sass paper_2206_11357_b200/libgact.so | awk -v pat="$1" '$0 ~ "Function : " {f = ($0 ~ pat)} f' \
  | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed -E 's@^\s+/\*([0-9a-f]+)\*/\s+@\1 @; s@\s*/\*.*@@' > /tmp/kernel.sass
echo "$(wc -l < /tmp/kernel.sass) instructions"
awk '{op=$2; if (op ~ /^@/) op=$3; sub(/\..*/, "", op); print op}' /tmp/kernel.sass | sort | uniq -c | sort -rn | head -${2:-25}
