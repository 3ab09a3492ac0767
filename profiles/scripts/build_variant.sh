#!/bin/bash
# Build a variant of the library with extra -D flags into scratch/var_<name>/ (for sweep.sh):
#   profiles/scripts/build_variant.sh minb2 -DSB_MTTKRP_MINB=2
set -e
cd "$(dirname "$0")/../.."
SRC=paper_1812_05961_b200/csrc
name=$1; shift
out=scratch/var_$name
mkdir -p $out
for f in $SRC/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -Iinclude "$@" -c $f -o $out/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsplatt_b200.so $out/*.o -ldl
rm -f $out/*.o
echo built $out
