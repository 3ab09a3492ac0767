# Sweep one environment variable ($VAR over $VALS) on c5 (or $CFG), two rounds, default first.
mkdir -p gpurun_out
P=${P:-sw}
for r in 1 2; do
  python bench.py --config ${CFG:-c5} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_def_$r.json 2> /dev/null
  for v in $VALS; do
    env $VAR=$v python bench.py --config ${CFG:-c5} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${P}_${v}_$r.json 2> /dev/null
  done
done
