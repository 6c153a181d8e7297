cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
LTFB_WIDE_V2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "stream or paper" > gpurun_out/w2k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w2k_pytest.log
tail -n 3 gpurun_out/w2k_pytest.log
LTFB_WIDE_V2=1 LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2k_bench20.json 2> gpurun_out/w2k_bench20.err; echo "bench20 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2k_bench20.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms_per_launch']['wide'], d['stream_profile_us'])"
grep -A 30 "stream prof" gpurun_out/w2k_bench20.err | tail -14 | head -13
grep "stream prof" gpurun_out/w2k_bench20.err | tail -1 | cut -c1-700
LTFB_WIDE_V2=1 timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/w2k_bench300.json 2> gpurun_out/w2k_bench300.err; echo "bench300 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2k_bench300.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'])"
