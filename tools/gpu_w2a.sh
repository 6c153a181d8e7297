# k_wide2 (64-column tiles): GPU suite, then bench (stream stage profile), launched-mode timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/w2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w2a_pytest.log
tail -n 30 gpurun_out/w2a_pytest.log
LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/w2a_bench20.json 2> gpurun_out/w2a_bench20.err; echo "bench20 rc=$?"; tail -c 1500 gpurun_out/w2a_bench20.json; grep -A 20 "stream prof" gpurun_out/w2a_bench20.err | tail -22
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/w2a_bench200.json 2> gpurun_out/w2a_bench200.err; echo "bench200 rc=$?"; tail -c 1200 gpurun_out/w2a_bench200.json
