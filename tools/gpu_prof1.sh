# stream stage profile with per-CTA phase-end stamps
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/prof1.json 2> gpurun_out/prof1.txt; echo rc=$?
grep "phase-2 barrier (us" gpurun_out/prof1.txt | head -8
