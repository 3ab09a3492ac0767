mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "csf or root2 or tiling" > gpurun_out/t_csf.log 2>&1; echo csf rc=$?; tail -3 gpurun_out/t_csf.log
SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/trace_c5.json 2> gpurun_out/trace_c5.err; echo trace rc=$?
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; echo bench rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_gpu.log 2>&1; echo gpu rc=$?; tail -3 gpurun_out/t_gpu.log
