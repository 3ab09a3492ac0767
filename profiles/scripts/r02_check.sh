mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; echo bench rc=$?
SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/trace_c5.json 2> gpurun_out/trace_c5.err; echo trace rc=$?
SPLATT_TRACE=1 python bench.py --config c3 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/trace_c3.json 2> gpurun_out/trace_c3.err; echo trace3 rc=$?
