mkdir -p gpurun_out
P=${P:-fc}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${P}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${P}_pytest.log
python bench.py > gpurun_out/${P}_bench_c5.json 2> gpurun_out/${P}_bench_c5.err
