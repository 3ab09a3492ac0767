mkdir -p gpurun_out
for r in 1 2; do
  for v in 1 2 3; do SPLATT_ROOT2_HOT=$v python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/hk_${v}_$r.json 2>/dev/null; done
  for b in b52 b40; do SPLATT_B200_LIB=scratch/var_$b/libsplatt_b200.so python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/hk_${b}_$r.json 2>/dev/null; done
done
