cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export LTFB_PARITY_REPORT=$PWD/gpurun_out/r2a_parity_report.jsonl
rm -f $LTFB_PARITY_REPORT
timeout 1800 python -m pytest tests -m gpu -q -k "not paper_k2" -p no:cacheprovider -rf > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench20.json 2> gpurun_out/r2a_bench20.err
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench1000.json 2> gpurun_out/r2a_bench1000.err
tail -3 gpurun_out/r2a_pytest.log; tail -2 gpurun_out/r2a_smoke.log
