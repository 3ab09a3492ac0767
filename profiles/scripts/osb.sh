mkdir -p gpurun_out
cd profiles/ab_r02 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 onesweep_bench.cu -o /tmp/osb && timeout 600 /tmp/osb 150000000 2>&1 | tee ../../gpurun_out/osb.txt
