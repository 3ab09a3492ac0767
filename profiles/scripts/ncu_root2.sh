mkdir -p gpurun_out
P=${P:-r2e}
for cfg in ${CFGS:-c5 c2}; do
python bench.py --config $cfg --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_plain_$cfg.json 2> gpurun_out/${P}_plain_$cfg.err && \
ncu --set full --clock-control none --import-source on -k regex:${KREG:-root2} -s ${SKIP:-5} -c 1 -o gpurun_out/${P}_$cfg python bench.py --config $cfg --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_$cfg.log 2>&1
done
