#!/bin/bash
# Build the library from an alternative source tree (a copy of csrc with changes) into
# scratch/var_<name>/libsplatt_b200.so:  build_tree_variant.sh <name> <csrc-dir> [-Dflags]
set -e
cd "$(dirname "$0")/../.."
name=$1; src=$2; shift 2
out=scratch/var_$name
mkdir -p $out
for f in $src/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -Iinclude "$@" -c $f -o $out/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsplatt_b200.so $out/*.o -ldl
rm -f $out/*.o
echo built $out
