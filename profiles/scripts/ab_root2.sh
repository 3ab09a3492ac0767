mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_determinism.py tests/test_gpu_policies.py tests/test_gpu_ridge.py -x -q -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2b_pytest.log
for cfg in c5 c2 c3 c4; do
  python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2b_${cfg}_v2.json 2> gpurun_out/r2b_${cfg}_v2.err
  SPLATT_ROOT2=0 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2b_${cfg}_v1.json 2> gpurun_out/r2b_${cfg}_v1.err
done
