# Round-2 final evidence: GPU tests, smoke, bench lines (c5 default with cpu_baseline/e2e, c3, c2),
# reference arm, ROOT MTTKRP DRAM traffic (c5, c3, c2), the c5 launch list, one full ncu capture.
mkdir -p gpurun_out
P=${P:-fin}
# SKIP_TESTS=1: the GPU test log comes from a separate call of the same tree
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/${P}_gpu_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_gpu_pytest.log
fi
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_smoke.log
python bench.py > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
python bench.py --config c3 --no-cpu-baseline > gpurun_out/${P}_bench_c3.json 2> gpurun_out/${P}_bench_c3.err
python bench.py --config c2 --no-cpu-baseline > gpurun_out/${P}_bench_c2.json 2> gpurun_out/${P}_bench_c2.err
python bench.py --impl reference > gpurun_out/${P}_reference_c5.json 2> gpurun_out/${P}_reference_c5.err
B="python bench.py --steps 1 --warmup 0 --iters 3 --no-cpu-baseline --no-e2e"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum
for cfg in c5 c2; do
  $B --config $cfg > gpurun_out/${P}_plain_$cfg.json 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:mttkrp -s 4 -c 8 --csv --log-file gpurun_out/${P}_traffic_$cfg.csv $B --config $cfg > gpurun_out/${P}_traffic_$cfg.log 2>&1
done
B3="python bench.py --steps 1 --warmup 0 --iters 10 --no-cpu-baseline --no-e2e --config c3"
$B3 > gpurun_out/${P}_plain_c3.json 2>&1 && \
ncu --metrics $M --clock-control none -k regex:mttkrp -s 20 -c 10 --csv --log-file gpurun_out/${P}_traffic_c3.csv $B3 > gpurun_out/${P}_traffic_c3.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --clocks off > gpurun_out/${P}_plain_launch.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_c5_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --clocks off > gpurun_out/${P}_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:root2 -s 5 -c 1 -o gpurun_out/${P}_root2_c5 $B --config c5 > gpurun_out/${P}_full.log 2>&1
echo done
