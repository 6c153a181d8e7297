# k_wide2 default: full GPU suite, smoke, bench 20 / default, launch list, ncu --set full of k_wide2 (launched)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/w2l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w2l_pytest.log
tail -n 6 gpurun_out/w2l_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/w2l_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/w2l_smoke.log
LTFB_STREAM_PROF=1 timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/w2l_bench20.json 2> gpurun_out/w2l_bench20.err; echo "bench20 rc=$?"
grep -A 8 "stream prof" gpurun_out/w2l_bench20.err | tail -8
timeout 600 python bench.py > gpurun_out/w2l_bench.json 2> gpurun_out/w2l_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2l_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['round_ms'], d['roofline']['frac'], d['kernel_rooflines']['wide'], d['stream_profile_us'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/w2l_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ae > gpurun_out/w2l_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
LTFB_NO_STREAM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide2 --launch-skip 4 -c 1 -o gpurun_out/w2l_wide2 python tools/step_driver.py --steps 8 > gpurun_out/w2l_ncu.log 2>&1; echo "ncu full rc=$?"
