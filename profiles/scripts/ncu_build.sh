mkdir -p gpurun_out
B="python bench.py --config c5 --steps 1 --warmup 1 --iters 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/nb_plain.json 2>&1; echo plain rc=$?
for spec in "downsweep_kernel:3" "level_write_kernel:1" "gather_kv_kernel:1" "decode_kernel:1" "upsweep_kernel:3" "level_count_kernel:1"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/nb_$k $B > gpurun_out/nb_$k.log 2>&1; echo $k rc=$?
done
