#!/bin/bash
# Build an A/B variant of the product library: tools/build_variant.sh NAME "NVCC FLAGS"
# -> paper_2604_14650_b200/lib/libNAME.so (objects in build/obj_NAME); select it at run
# time with LPM6CU_LIB=paper_2604_14650_b200/lib/libNAME.so (tools/ab_bench.sh).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -j"$(nproc)" -C "$ROOT/paper_2604_14650_b200/csrc" OBJDIR="$ROOT/build/obj_$1" LIBNAME="lib$1.so" EXTRA_NVFLAGS="$2" >/dev/null
echo "built paper_2604_14650_b200/lib/lib$1.so ($2)"
