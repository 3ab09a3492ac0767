mkdir -p gpurun_out
(cd profiles/ab_r02 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 onesweep_bench.cu -o /tmp/osb && timeout 600 /tmp/osb 150000000 > ../../gpurun_out/osb.txt 2>&1)
for g in 32 64 default; do
  if [ $g = default ]; then unset SPLATT_L2_FETCH; else export SPLATT_L2_FETCH=$g; fi
  SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/l2f_trace_$g.json 2> gpurun_out/l2f_trace_$g.err
  python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l2f_c5_$g.json 2> gpurun_out/l2f_c5_$g.err; echo $g rc=$?
done
