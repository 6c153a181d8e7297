# Launch list of the bench command (the streamed step turns itself off under
# ncu via the concurrency probe), smoke under ncu, and a streamed bench check.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f2_bench20.json 2> gpurun_out/f2_bench20.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --rounds 2 --e2e-steps 2 > gpurun_out/f2_ncu_launch.log 2>&1; echo "ncu launch rc=$?" >> gpurun_out/f2_ncu_launch.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke_ncu.log 2>&1; echo "smoke ncu rc=$?" >> gpurun_out/f2_smoke_ncu.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "stream or bench_contract or smoke" > gpurun_out/f2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f2_pytest.log
tail -n 2 gpurun_out/f2_ncu_launch.log gpurun_out/f2_smoke_ncu.log gpurun_out/f2_pytest.log
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/f2_bench20.json").read().splitlines() if l.startswith("{")][-1])
print(d.get("value"), d.get("ms_per_step"), d.get("step_mode"), d.get("gpu_launches"), (d.get("e2e") or {}).get("value"))
PY
