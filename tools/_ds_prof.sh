cd $GRAFT_REPO_ROOT
FGFRFT_SYN_CAP0=40 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dsynth_kernel -c 1 -o gpurun_out/ds40 python tools/c3_step.py --steps 1 --warmup 1 > gpurun_out/ds_ncu.log 2>&1
tail -2 gpurun_out/ds_ncu.log
