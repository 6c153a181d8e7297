# k_wide2 with 32-B epilogue loads: quick parity subset, bench (stream profile), ncu --set full of the launched kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "stream or paper" > gpurun_out/w2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w2b_pytest.log
tail -n 3 gpurun_out/w2b_pytest.log
LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/w2b_bench20.json 2> gpurun_out/w2b_bench20.err; echo "bench20 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2b_bench20.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms_per_launch'], d['stream_profile_us'])"
grep -A 20 "stream prof" gpurun_out/w2b_bench20.err | tail -22
LTFB_NO_STREAM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide2 --launch-skip 3 -c 1 -o gpurun_out/w2b_wide2 python tools/step_driver.py --steps 6 > gpurun_out/w2b_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/w2b_ncu.log
