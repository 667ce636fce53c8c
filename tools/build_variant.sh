#!/bin/bash
# Build an A/B variant of libepi3cu.so with extra nvcc defines into
# build/v_<name>/libepi3cu.so (select it with E3_LIBCU=... for tools/syrk_time.py).
#   tools/build_variant.sh prof -DE3_PROFILE_SKIP=1
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/build/v_$NAME
mkdir -p "$OUT"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include -I$ROOT/paper_2201_10956_b200/csrc"
$NVCC $FL "$@" -c "$ROOT/paper_2201_10956_b200/csrc/engine.cu" -o "$OUT/engine.o"
$NVCC $FL -c "$ROOT/paper_2201_10956_b200/csrc/host.cpp" -o "$OUT/host.o"
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libepi3cu.so" "$OUT/engine.o" "$OUT/host.o" -cudart shared
rm -f "$OUT/engine.o" "$OUT/host.o"  # keep the gpurun snapshot small (< 512 MiB)
echo "$OUT/libepi3cu.so"
