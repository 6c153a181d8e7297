# re-entry check: full GPU suite, smoke, bench (20 + default), AE bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l_pytest.log
tail -n 8 gpurun_out/l_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/l_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/l_bench20.json 2> gpurun_out/l_bench20.err; echo "bench20 rc=$?"; tail -c 3000 gpurun_out/l_bench20.json
timeout 600 python bench.py > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/l_bench.json
timeout 300 python tools/ae_bench.py --dims paper > gpurun_out/l_ae_paper.json 2>&1; cat gpurun_out/l_ae_paper.json | tail -2
