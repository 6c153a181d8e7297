cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LTFB_STREAM_PROF=1 timeout 120 python tools/stream_check.py --steps 8 --n 8000 --time-steps 200 > gpurun_out/r2e_prof.json 2> gpurun_out/r2e_prof.err
tail -n 6 gpurun_out/r2e_prof.err
