# Round-2 evidence on one B200: GPU tests, bench (both arms), configs, launch list of the bench
# command, ncu --set full of the config-3 step's kernels and the config-5 kernels. Outputs under
# gpurun_out/ev2/ (summaries copied into profiles/ by hand: tools/ncu_summary.py, tools/launch_table.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev2
E=gpurun_out/ev2
timeout 1500 python -m pytest tests -m gpu -q -x > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $E/pytest_gpu.log
tail -2 $E/pytest_gpu.log
timeout 600 python bench.py > $E/bench.json 2> $E/bench.err
timeout 600 python bench.py --impl reference > $E/bench_ref.json 2> $E/bench_ref.err
timeout 900 python tools/bench_configs.py --configs 1,2,3,4,5 > $E/configs.jsonl 2> $E/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $E/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $E/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"psynth|ozgemm_kernel|oz_slice|oz_rowslice|mse_dy" -s 8 -c 6 -o $E/prof_c3 python tools/c3_step.py --steps 2 --warmup 2 > $E/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"batch_fwd_tc|batch_dlda_tc" -s 4 -c 2 -o $E/prof_c5 python tools/bench_configs.py --configs 5 > $E/ncu_c5.log 2>&1
tail -c 400 $E/bench.json
