#!/bin/bash
# Final measurement pass: GPU tests, benches for every config, ncu launch list + captures,
# per-config DRAM traffic of the ROOT MTTKRP.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/f_gpu_tests.log 2>&1; echo tests=$?
timeout 400 python bench.py > $O/f_bench_c2.json 2> $O/f_bench_c2.err; echo c2=$?
for c in c3 c4 c4r64 c5; do timeout 700 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/f_bench_$c.json 2> $O/f_bench_$c.err; echo $c=$?; done
for p in one two; do timeout 400 python bench.py --policy $p --no-cpu-baseline --no-e2e > $O/f_bench_c2_$p.json 2> /dev/null; echo $p=$?; done
timeout 400 python bench.py --impl reference --steps 1 --warmup 0 > $O/f_ref_c2.json 2> $O/f_ref_c2.err; echo ref=$?
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/f_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --clocks off > /dev/null 2>&1; echo ncu1=$?
# --iters 5: the gather policy is timed on iterations 1-2, so launches 7.. run the chosen variant
timeout 700 ncu --set full --clock-control none --import-source on -k regex:mttkrp_csf_kernel -s 9 -c 3 -o $O/f_mttkrp_c2 python bench.py --steps 1 --warmup 0 --iters 5 --no-cpu-baseline --no-e2e --clocks off > /dev/null 2>&1; echo ncu2=$?
timeout 700 ncu --set full --clock-control none --import-source on -k regex:solve_gram -s 3 -c 3 -o $O/f_solve_c2 python bench.py --steps 1 --warmup 1 --iters 2 --no-cpu-baseline --no-e2e --clocks off > /dev/null 2>&1; echo ncu3=$?
timeout 700 ncu --set full --clock-control none --import-source on -k regex:mttkrp_csf_kernel -s 3 -c 3 -o $O/f_mttkrp_c2_one python bench.py --policy one --steps 1 --warmup 1 --iters 2 --no-cpu-baseline --no-e2e --clocks off > /dev/null 2>&1; echo ncu4=$?
for c in c4 c5; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --csv -k regex:mttkrp_csf_kernel -s 0 -c 8 --log-file $O/f_traffic_$c.csv python bench.py --config $c --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e --clocks off > /dev/null 2>&1; echo traffic_$c=$?
done
