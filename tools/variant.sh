#!/bin/bash
# Build a variant of the library with extra nvcc defines for same-box A/B:
#   tools/variant.sh NAME "-DAXL_X=1 -DAXL_Y=2" [source.cu ...]  ->  scratch/NAME/libaxhelm_sm100.so
# Only the listed sources (default: ax_line.cu axhelm.cu) are recompiled; the
# other objects are the tree's.
set -e
NAME=$1; DEFS=$2; shift 2; SRCS=${*:-ax_line.cu axhelm.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2506_20994_b200/csrc
W=/tmp/axvar_$NAME
rm -rf "$W"; mkdir -p "$W/pkg/csrc" "$W/include" "$ROOT/scratch/$NAME"
cp "$SRC"/*.cu "$SRC"/*.cuh "$SRC"/*.h "$SRC"/Makefile "$W/pkg/csrc/"
cp "$ROOT"/include/*.h "$W/include/"
mkdir -p "$W/pkg/csrc/build"; cp "$SRC"/build/*.o "$W/pkg/csrc/build/"
for f in $SRCS; do rm -f "$W/pkg/csrc/build/${f%.cu}.o"; done  # rebuilt for sure (no mtime races)
make -C "$W/pkg/csrc" -j4 NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v $DEFS" LIB="$ROOT/scratch/$NAME/libaxhelm_sm100.so" > "$W/make.log" 2>&1 || { tail -30 "$W/make.log"; exit 1; }
echo "built scratch/$NAME/libaxhelm_sm100.so"
