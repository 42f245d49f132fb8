cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_fwd_tc -s 2 -c 1 -o gpurun_out/c5fwd python tools/bench_configs.py --configs 5 > gpurun_out/ncu_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batch_dlda_tc -s 2 -c 1 -o gpurun_out/c5bwd python tools/bench_configs.py --configs 5 >> gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_c5.log
