# Round-end evidence on one B200: GPU tests, bench (both arms), configs, launch list, ncu full
# capture of the hot kernels. Outputs under gpurun_out/ev/ (copied into profiles/ by hand).
set -x
mkdir -p gpurun_out/ev
python -m pytest tests -m gpu -q -x > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev/pytest_gpu.log
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err
python bench.py --impl reference > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
python tools/bench_configs.py --configs 1,2,3,4,5 > gpurun_out/ev/configs_int8.jsonl 2> gpurun_out/ev/configs_int8.err
FGFRFT_ENGINE=dmma python tools/bench_configs.py --configs 2,3,4 > gpurun_out/ev/configs_dmma.jsonl 2> gpurun_out/ev/configs_dmma.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ev/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ozgemm_kernel|node_combine|rsynth|rapply_fused" -c 12 -o gpurun_out/ev/prof python tools/profile_kernels.py > gpurun_out/ev/ncu_full.log 2>&1
tail -2 gpurun_out/ev/pytest_gpu.log
ncu --set full --clock-control none --import-source on -k regex:"batch_forward|batch_dlda" -c 2 -o gpurun_out/ev/prof_c5 python tools/bench_configs.py --configs 5 > gpurun_out/ev/ncu_c5.log 2>&1
