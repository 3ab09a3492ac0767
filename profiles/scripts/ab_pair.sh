# A/B: scratch/var_$A (SPLATT_B200_LIB) against the in-tree library, alternating, c5 by default.
mkdir -p gpurun_out
P=${P:-ab}
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "$TESTS" > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log; fi
for r in 1 2; do
  for cfg in ${CFGS:-c5}; do
    SPLATT_B200_LIB=scratch/var_$A/libsplatt_b200.so python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_base$r.json 2> gpurun_out/${P}_${cfg}_base$r.err
    python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_new$r.json 2> gpurun_out/${P}_${cfg}_new$r.err
  done
done
