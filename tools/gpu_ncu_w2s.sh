# ncu --set full with source counters of the launched k_wide2 (paper dims)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LTFB_NO_STREAM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide2 --launch-skip 3 -c 1 -o gpurun_out/w2s_wide2 python tools/step_driver.py --steps 6 > gpurun_out/w2s_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/w2s_ncu.log
