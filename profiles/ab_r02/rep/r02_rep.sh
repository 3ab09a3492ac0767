# Hot rows in per-CTA global replicas (SB_ROOT2_REP=1, scratch/var_rep) vs the shared-memory table:
# parity of the 4-mode kernel with the variant, then c5 MTTKRP per launch over K.
mkdir -p gpurun_out
P=${P:-rep}
L=scratch/var_rep/libsplatt_b200.so
for k in 2 64; do
  SPLATT_B200_LIB=$L SPLATT_ROOT2_HOT=$k timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "root2 or four_mode" > gpurun_out/${P}_pytest_k$k.log 2>&1; echo rc=$? >> gpurun_out/${P}_pytest_k$k.log
done
B="python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for r in 1 2; do
  $B > gpurun_out/${P}_base_$r.json 2>/dev/null
  for k in ${KS:-2 8 32 128 512}; do
    SPLATT_B200_LIB=$L SPLATT_ROOT2_HOT=$k $B > gpurun_out/${P}_k${k}_$r.json 2>/dev/null
  done
done
