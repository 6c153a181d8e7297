cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for S in 130 128 132; do
LTFB_WIDE_CTAS=$S LTFB_STREAM_PROF=2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2p_$S.json 2> gpurun_out/w2p_$S.err; echo "S=$S prof rc=$?"
grep "per CTA step" gpurun_out/w2p_$S.err | head -5
grep -A 3 "stream prof" gpurun_out/w2p_$S.err | grep "partials per CTA" | head -2
LTFB_WIDE_CTAS=$S timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/w2p_b$S.json 2> gpurun_out/w2p_b$S.err; python -c "
import json; d=json.loads(open('gpurun_out/w2p_b$S.json').read().strip().splitlines()[-1]); print('S=$S', d['ms_per_step'], d['value'], d['stream_profile_us']['step_us'], d['stream_profile_us']['h_to_phase2_reduced_us'])"
done
