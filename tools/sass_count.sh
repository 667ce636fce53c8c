#!/bin/bash
# Instruction count of each search_syrk_kernel instantiation of a library build
# (template args <kRanged, kMode, kSS>), for A/B of code size before GPU time.
#   tools/sass_count.sh paper_2201_10956_b200/libepi3cu.so
LIB=$(readlink -f "$1")
d=$(mktemp -d); cd "$d" || exit 1
cuobjdump -xelf all "$LIB" >/dev/null 2>&1
cuobjdump -sass engine.sm_100a.cubin 2>/dev/null | awk '
  /Function : /{ if (name != "") print name, n; name = ""; n = 0
                 if ($3 ~ /search_syrk_kernel/) { name = $3; sub(/.*kernelI/, "", name); sub(/EEvN.*/, "", name) } next }
  name != "" && /\/\*[0-9a-f]+\*\/ / { n++ }
  END { if (name != "") print name, n }'
cd / && rm -rf "$d"
