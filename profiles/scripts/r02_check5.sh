mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "csf" > gpurun_out/t_csf.log 2>&1; echo csf rc=$?; tail -1 gpurun_out/t_csf.log
SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/trace_c5.json 2> gpurun_out/trace_c5.err
