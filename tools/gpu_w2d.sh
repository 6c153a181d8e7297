cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/w2_trunc_check.py > gpurun_out/w2d_trunc.json 2>&1; echo "trunc rc=$?"; tail -2 gpurun_out/w2d_trunc.json
LTFB_STREAM_PROF=2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/w2d_bench20.json 2> gpurun_out/w2d_bench20.err; echo "bench20 rc=$?"
grep -A 4 "stream prof" gpurun_out/w2d_bench20.err | grep "per CTA" | tail -1 > gpurun_out/w2d_percta.txt; wc -c gpurun_out/w2d_percta.txt
