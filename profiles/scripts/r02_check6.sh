mkdir -p gpurun_out
for r in 1 2; do
SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/tr_new$r.json 2> gpurun_out/tr_new$r.err
SPLATT_B200_LIB=scratch/var_noldg/libsplatt_b200.so SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/tr_old$r.json 2> gpurun_out/tr_old$r.err
done
