# A/B of one environment setting ($ENVAB, e.g. SPLATT_ROOT2_WIDE=1) against the default, same
# library, alternating, c5 by default; $TESTS: pytest -k filter run with the setting first.
mkdir -p gpurun_out
P=${P:-abenv}
if [ -n "$TESTS" ]; then env $ENVAB timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "$TESTS" > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log; fi
for r in 1 2; do
  for cfg in ${CFGS:-c5}; do
    python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_base$r.json 2> gpurun_out/${P}_${cfg}_base$r.err
    env $ENVAB python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_new$r.json 2> gpurun_out/${P}_${cfg}_new$r.err
  done
done
