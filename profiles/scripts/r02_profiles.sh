# Round-2 evidence: DRAM traffic / L2 hit / L1TEX load per ROOT MTTKRP launch (c5, c3, c2),
# the c5 launch list, and one --set full capture of the c5 ROOT kernel.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --iters 3 --no-cpu-baseline --no-e2e"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum
for cfg in c5 c3 c2; do
  $B --config $cfg > gpurun_out/r02p_plain_$cfg.json 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:mttkrp -s 4 -c 8 --csv --log-file gpurun_out/r02p_traffic_$cfg.csv $B --config $cfg > gpurun_out/r02p_traffic_$cfg.log 2>&1
done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --clocks off > gpurun_out/r02p_plain_launch.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02p_c5_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --clocks off > gpurun_out/r02p_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:root2 -s 5 -c 1 -o gpurun_out/r02p_root2_c5 $B --config c5 > gpurun_out/r02p_full.log 2>&1
