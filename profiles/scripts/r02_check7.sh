mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_policies.py -x -q -k "csf or root2 or tiling or policy or policies" > gpurun_out/t_csf.log 2>&1; echo csf rc=$?; tail -1 gpurun_out/t_csf.log
for r in 1 2; do
SPLATT_TRACE=1 python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e > gpurun_out/tr_lw$r.json 2> gpurun_out/tr_lw$r.err
done
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
