#!/bin/bash
# Build a tuning variant of libtmop_b200.so into variants/<name>/ :
#   tools/build_variant.sh <name> "-DTMOP_ELEM_NT=128 -DTMOP_SMEM_BUDGET=7168 -DTMOP_MIN_BLOCKS=4"
# Select it at run time with TMOP_LIB=vlibs/<name>/libtmop_b200.so.
set -e
name=$1; defs=$2
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/vlibs/$name; obj=$root/build/variants/$name
mkdir -p "$out" "$obj"
cd "$root/paper_2205_12721_b200/csrc"
make -s -j8 OUT="$out/libtmop_b200.so" OBJDIR="$obj" NVCC="nvcc $defs" all
echo "$out/libtmop_b200.so"
