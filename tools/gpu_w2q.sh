cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for R in 0 5; do
LTFB_W2_ROT=$R LTFB_STREAM_PROF=2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2q_$R.json 2> gpurun_out/w2q_$R.err; echo "rot=$R rc=$?"
grep "per CTA step" gpurun_out/w2q_$R.err | head -5
done
