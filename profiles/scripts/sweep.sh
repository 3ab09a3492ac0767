#!/bin/bash
# usage: sweep.sh config iters -> one line per variant with MTTKRP nnz.R/s
cfg=$1; it=$2
for d in paper_1812_05961_b200 scratch/var_*; do
  lib=$d/libsplatt_b200.so
  r=$(SPLATT_B200_LIB=$lib timeout 300 python bench.py --config $cfg --iters $it --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --clocks off 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.4e %.3f %.2f' % (d['mttkrp_nnzR_per_s'], d['roofline']['frac'], d['ms_per_step']))")
  echo "$cfg $(basename $d) $r"
done
