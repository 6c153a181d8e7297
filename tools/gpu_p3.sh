# post: dec-head backward in the D/G half (no S3b), S6 arrive-only + DSMEM pull of the new fwd
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/p3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p3_pytest.log
tail -n 3 gpurun_out/p3_pytest.log
for i in 1 2; do
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/p3_bench20_$i.json 2> gpurun_out/p3_bench20_$i.err; echo "bench20 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/p3_bench20_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['stream_profile_us'])"
done
LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/p3_prof.json 2> gpurun_out/p3_prof.err; echo "prof rc=$?"
grep -A 14 "stream prof" gpurun_out/p3_prof.err | tail -14 | head -6
grep "stream prof" gpurun_out/p3_prof.err | tail -1 | cut -c1-800
