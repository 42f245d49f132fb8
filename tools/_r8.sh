cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev2
E=gpurun_out/ev2
timeout 600 python tools/probe_c2_after_c3.py > $E/probe_c2.log 2>&1
cat $E/probe_c2.log | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $E/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $E/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"psynth|ozgemm_kernel<6, 1|mse_dy|oz_slice_direct_kernel<6>|oz_rowslice_pairs_kernel<6>" -s 6 -c 6 -o $E/prof_c3 python tools/c3_step.py --steps 2 --warmup 2 > $E/ncu_c3.log 2>&1
tail -2 $E/ncu_c3.log
