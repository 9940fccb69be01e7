#!/bin/bash
# Code size (instructions) per source line of one kernel in a cubin:
#   tools/sass_size.sh <cubin> <mangled-kernel-name> [top]
nvdisasm -g "$1" 2>/dev/null | awk -v fn="$2" '
  /^\/\/-+ \.text\./ { on = index($0, ".text." fn " ") > 0; next }
  on && /\/\/## File/ { match($0, /line [0-9]+/); split($0, x, "\""); f = x[2]; sub(/.*\//, "", f);
                        key = f ":" substr($0, RSTART + 5, RLENGTH - 5) }
  on && /\/\*[0-9a-f]{4}\*\// { c[key]++; tot++ }
  END { print tot, "instructions"; for (k in c) print c[k], k }' | sort -rn | head -${3:-30}
