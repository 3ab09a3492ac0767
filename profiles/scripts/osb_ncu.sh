mkdir -p gpurun_out
cd profiles/ab_r02 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo onesweep_bench.cu -o /tmp/osb && \
timeout 600 /tmp/osb 150000000 > ../../gpurun_out/osb.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:onesweep_kernel -s 5 -c 1 -o ../../gpurun_out/osb_p256x12 /tmp/osb 150000000 > ../../gpurun_out/osb_ncu.log 2>&1
