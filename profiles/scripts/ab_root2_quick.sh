mkdir -p gpurun_out
P=${P:-r2d}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "mttkrp or root_kernel" > gpurun_out/${P}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${P}_pytest.log
for cfg in ${CFGS:-c5 c2}; do
  python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_v2.json 2> gpurun_out/${P}_${cfg}_v2.err
  if [ -n "$NOHOT" ]; then SPLATT_ROOT2_HOT=0 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_v2nohot.json 2> gpurun_out/${P}_${cfg}_v2nohot.err; fi
  if [ -n "$V1" ]; then SPLATT_ROOT2=0 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${cfg}_v1.json 2> gpurun_out/${P}_${cfg}_v1.err; fi
done
