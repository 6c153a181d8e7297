cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export LTFB_PARITY_REPORT=$PWD/gpurun_out/r2g_parity_report.jsonl
rm -f $LTFB_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2g_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench20.json 2> gpurun_out/r2g_bench20.err
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/r2g_bench1000.json 2> gpurun_out/r2g_bench1000.err
tail -4 gpurun_out/r2g_pytest.log; tail -2 gpurun_out/r2g_smoke.log
python -c "
import json
for f in ('gpurun_out/r2g_bench20.json','gpurun_out/r2g_bench1000.json'):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['ms_per_step'], d['round_ms'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])
    except Exception as e: print(f, 'failed', e)
"
tail -3 gpurun_out/r2g_bench20.err
