# Round-2 measurement set on one B200 (results copied into profiles/ by hand)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export LTFB_PARITY_REPORT=$PWD/gpurun_out/f1_parity_report.jsonl
rm -f $LTFB_PARITY_REPORT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/f1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f1_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f1_ref.json 2> gpurun_out/f1_ref.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f1_bench20.json 2> gpurun_out/f1_bench20.err
timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/f1_bench1000.json 2> gpurun_out/f1_bench1000.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f1_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --rounds 2 --e2e-steps 2 > gpurun_out/f1_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_wide_tc|k_post_small|k_eval_tc" -s 12 -c 3 -o gpurun_out/f1_full python bench.py --steps 20 --warmup 3 --no-cpu-baseline --rounds 2 --e2e-steps 2 > gpurun_out/f1_ncu_full.log 2>&1
tail -3 gpurun_out/f1_pytest.log; tail -1 gpurun_out/f1_smoke.log
python - <<'PY'
import json
for f in ("f1_ref.json","f1_bench20.json","f1_bench1000.json"):
    try:
        d=json.loads([l for l in open("gpurun_out/"+f).read().splitlines() if l.startswith("{")][-1])
        print(f, d.get("value"), d.get("ms_per_step"), d.get("round_ms"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("stream_profile_us"))
    except Exception as e: print(f, "failed", e)
PY
ls -la gpurun_out/f1_full* 2>/dev/null; tail -2 gpurun_out/f1_ncu_full.log
