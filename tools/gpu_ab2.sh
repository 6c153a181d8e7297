# A/B: tile rotation (stragglers on CTAs 16/17 get 5 tiles), and desk dims k_wide2 vs the 32-column kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3; do for R in 0 100; do
LTFB_W2_ROT=$R timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ae 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('rot=$R', round(d['ms_per_step']*1000,2), d['stream_profile_us'].get('step_us'), d['stream_profile_us'].get('h_to_phase2_reduced_us'))"
done; done
LTFB_W2_ROT=100 LTFB_STREAM_PROF=2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/ab2_prof.json 2> gpurun_out/ab2_prof.err; grep "per CTA step" gpurun_out/ab2_prof.err | head -4
for v in 0 1; do
if [ $v = 1 ]; then export LTFB_WIDE_V1=1; else unset LTFB_WIDE_V1; fi
timeout 300 python bench.py --dims desk --samples-per-trainer 60000 --steps 40 --warmup 5 --no-cpu-baseline --no-ae 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('desk V1=$v', round(d['ms_per_step']*1000,2), d['value'], d['config']['wide_ctas'], d['stream_profile_us'].get('step_us'))"
done
