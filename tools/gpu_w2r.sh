cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/w2r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w2r_pytest.log
tail -n 3 gpurun_out/w2r_pytest.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/w2r_bench20.json 2> gpurun_out/w2r_bench20.err; echo "bench20 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2r_bench20.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['kernels_ms_per_launch'], d['kernel_rooflines']['wide']['frac'], d['stream_profile_us']['step_us'])"
