# Round-2 closing evidence at HEAD on one B200 (after the side-stream / host-step changes): outputs under gpurun_out/ev11/.
cd $GRAFT_REPO_ROOT
E=gpurun_out/ev11; mkdir -p $E
timeout 1800 python -m pytest tests -m gpu -q -x > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $E/pytest_gpu.log
tail -n 2 $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; tail -n 1 $E/smoke.log
timeout 900 python bench.py > $E/bench.json 2> $E/bench.err; tail -c 200 $E/bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $E/bench_ref.json 2> $E/bench_ref.err
timeout 600 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > $E/bench_sharded.json 2> $E/bench_sharded.err; tail -c 300 $E/bench_sharded.json
timeout 900 python tools/bench_configs.py --configs 1,2,3,4,5 > $E/configs.jsonl 2> $E/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $E/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $E/ncu_bench.log 2>&1
ls $E
