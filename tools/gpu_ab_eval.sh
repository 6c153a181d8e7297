# eval kernel A/B: parity subset + round time (bench round_ms) interleaved
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/abe_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/abe_pytest.log
tail -n 2 gpurun_out/abe_pytest.log
for i in 1 2 3; do for v in base new; do
LTFB_LIB_PATH=$PWD/tools/ab/lib_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ae 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['ms_per_step']*1000,2), 'round_ms', round(d['round_ms'],4))"
done; done
for v in base new; do LTFB_LIB_PATH=$PWD/tools/ab/lib_$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_eval_tc --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ae 2>/dev/null | grep k_eval_tc | awk -F, -v v=$v '{gsub(/"/,"",$NF); s+=$NF; n++} END {print v, "k_eval_tc us", s/n/1000, n}'; done
