# A/B: specialised post routines (-DLTFB_POST_SPECIALIZE) vs runtime-shaped
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3; do for v in base new; do
LTFB_LIB_PATH=$PWD/tools/ab/lib_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ae 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['ms_per_step']*1000,2), d['stream_profile_us'].get('step_us'), d['stream_profile_us'].get('post_chain_after_dec_us'), d['stream_profile_us'].get('d_step_overlapped_us'), round(d['kernels_ms_per_launch']['post']*1000,2))"
done; done
