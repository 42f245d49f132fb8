cd $GRAFT_REPO_ROOT
E=gpurun_out/ev7; mkdir -p $E
timeout 1800 python -m pytest tests -m gpu -q -x > $E/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $E/pytest_gpu.log
tail -n 2 $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; tail -n 1 $E/smoke.log
timeout 900 python bench.py > $E/bench.json 2> $E/bench.err; tail -c 300 $E/bench.json
