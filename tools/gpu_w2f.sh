cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in 0 2 4 8 14; do
LTFB_WIDE_V2=1 LTFB_W2_FLAGS=$f LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2f_$f.json 2> gpurun_out/w2f_$f.err; echo "flags=$f rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2f_$f.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms_per_launch']['wide'], d['stream_profile_us'])"
grep -A 30 "stream prof" gpurun_out/w2f_$f.err | tail -12
done
