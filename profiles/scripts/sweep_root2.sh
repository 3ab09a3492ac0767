# usage: P=prefix CFGS="c5" VARS="t384u3 ..." CHUNKS="512 2048" bash profiles/scripts/sweep_root2.sh
mkdir -p gpurun_out
P=${P:-sw}
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for cfg in ${CFGS:-c5}; do
  $B --config $cfg > gpurun_out/${P}_${cfg}_base.json 2> gpurun_out/${P}_${cfg}_base.err
  for v in $VARS; do
    SPLATT_B200_LIB=scratch/var_$v/libsplatt_b200.so $B --config $cfg > gpurun_out/${P}_${cfg}_$v.json 2> gpurun_out/${P}_${cfg}_$v.err
  done
  for ch in $CHUNKS; do
    SPLATT_CHUNK=$ch $B --config $cfg > gpurun_out/${P}_${cfg}_ch$ch.json 2> gpurun_out/${P}_${cfg}_ch$ch.err
  done
done
