cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
LTFB_WIDE_V2=1 LTFB_STREAM_PROF=2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2i_$i.json 2> gpurun_out/w2i_$i.err; echo "rc=$?"
done
