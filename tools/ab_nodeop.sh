mkdir -p gpurun_out/ab
for v in 1 0; do
FGFRFT_NODE_FUSED_ROWMAX=$v python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab/bench_$v.json 2>/dev/null
FGFRFT_NODE_FUSED_ROWMAX=$v ncu --set full --clock-control none --import-source on -k regex:ozgemm -c 1 -o gpurun_out/ab/nodeop_$v python tools/profile_kernels.py > gpurun_out/ab/ncu_$v.log 2>&1
done
