# Round-2 (fourth session, final) evidence at HEAD on one B200: outputs under gpurun_out/ev10/ (summaries copied to profiles/).
cd $GRAFT_REPO_ROOT
E=gpurun_out/ev10; mkdir -p $E
timeout 1800 python -m pytest tests -m gpu -q -x > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $E/pytest_gpu.log
tail -n 2 $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; tail -n 1 $E/smoke.log
timeout 900 python bench.py > $E/bench.json 2> $E/bench.err; tail -c 200 $E/bench.json
timeout 600 python bench.py --impl reference > $E/bench_ref.json 2> $E/bench_ref.err
timeout 600 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > $E/bench_sharded.json 2> $E/bench_sharded.err; tail -c 300 $E/bench_sharded.json
timeout 900 python tools/bench_configs.py --configs 1,2,3,4,5 > $E/configs.jsonl 2> $E/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $E/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $E/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:psynth|prow_bound|ozgemm_kernel<\(int\)6, \(int\)1|fused_mse|oz_rowslice_pairs_kernel<\(int\)6>" -s 6 -c 5 -o $E/prof_c3 python tools/c3_step.py --steps 2 --warmup 2 > $E/ncu_c3.log 2>&1
ls $E
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:ozgemm_kernel<\(int\)6, \(int\)0|node_combine|oz_slice_direct_kernel<\(int\)6>" -s 8 -c 3 -o $E/prof_c2 python tools/probe_regress.py c2 > $E/ncu_c2.log 2>&1
PROBE_TRACE=1 timeout 300 python tools/probe_regress.py c2 > $E/c2_trace.jsonl 2>&1
timeout 900 python tools/c3_step.py --config 4 --steps 10 --warmup 3 > $E/c4_step.json 2> $E/c4_step.err
ls $E
