mkdir -p gpurun_out
for r in 1 2; do
  python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/la_def_$r.json 2>/dev/null
  for b in l1a46 l1a48; do SPLATT_B200_LIB=scratch/var_$b/libsplatt_b200.so python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/la_${b}_$r.json 2>/dev/null; done
done
