#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { r=$(SPLATT_CHUNK=$2 timeout 300 python bench.py --config $1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --clocks off 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.4e %.2f' % (d['mttkrp_nnzR_per_s'], d['ms_per_step']))"); echo "$1 chunk=$2 $r"; }
for ch in default 192 224 256 288 320; do run c2 $ch; done
for ch in default 384 512 640 768; do run c4 $ch; done
