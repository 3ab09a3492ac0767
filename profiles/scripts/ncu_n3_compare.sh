# ncu of the 3-mode ROOT kernels on c2: first generation (default) vs second (SPLATT_ROOT2=3)
mkdir -p gpurun_out
B="python bench.py --config c2 --steps 1 --warmup 0 --iters 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/n3c_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mttkrp -s 4 -c 1 -o gpurun_out/n3c_v1 $B > gpurun_out/n3c_v1.log 2>&1
SPLATT_ROOT2=3 $B > gpurun_out/n3c_plain2.json 2>&1 && \
SPLATT_ROOT2=3 ncu --set full --clock-control none --import-source on -k regex:mttkrp -s 4 -c 1 -o gpurun_out/n3c_v2 $B > gpurun_out/n3c_v2.log 2>&1
