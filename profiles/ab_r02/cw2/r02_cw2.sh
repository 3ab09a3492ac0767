# ROOT v2 (4-mode) with two columns per lane (SB_ROOT2_CW=2: 16-byte gathers, 8-lane groups at
# R = 16, 80 registers) at 512/640/768/1024 threads vs the default (4 columns, 512 threads).
mkdir -p gpurun_out
P=${P:-cw2}
SPLATT_B200_LIB=scratch/var_cw2t768/libsplatt_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "root2 or four_mode or mttkrp" > gpurun_out/${P}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${P}_pytest.log
B="python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for r in 1 2; do
  $B > gpurun_out/${P}_base_$r.json 2>/dev/null
  for v in ${VARS:-cw2t768 cw2t512 cw2t640 cw2t1024}; do
    SPLATT_B200_LIB=scratch/var_$v/libsplatt_b200.so $B > gpurun_out/${P}_${v}_$r.json 2>/dev/null
  done
done
