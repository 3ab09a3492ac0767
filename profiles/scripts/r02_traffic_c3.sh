mkdir -p gpurun_out
B="python bench.py --config c3 --steps 1 --warmup 0 --iters 10 --no-cpu-baseline --no-e2e"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum
$B > gpurun_out/r02p_plain_c3t.json 2>&1 && \
ncu --metrics $M --clock-control none -k regex:mttkrp -s 20 -c 10 --csv --log-file gpurun_out/r02p_traffic_c3t.csv $B > gpurun_out/r02p_traffic_c3t.log 2>&1
