cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LTFB_STREAM_PROF=2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2o_prof.json 2> gpurun_out/w2o_prof.err; echo "prof rc=$?"
grep "per CTA step" gpurun_out/w2o_prof.err | head -30
