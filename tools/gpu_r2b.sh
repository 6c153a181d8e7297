cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export LTFB_PARITY_REPORT=$PWD/gpurun_out/r2b_parity_report.jsonl
rm -f $LTFB_PARITY_REPORT
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "run_experiment or state_injection" > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
for tool in memcheck synccheck racecheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2b_sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_sanitize_$tool.log
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control all -k regex:"k_wide_tc|k_post_small|k_eval_tc" -s 30 -c 6 --csv --log-file gpurun_out/r2b_traffic_cold.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --rounds 2 --e2e-steps 2 > gpurun_out/r2b_ncu_cold.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:"k_wide_tc|k_post_small|k_eval_tc" -s 30 -c 6 --csv --log-file gpurun_out/r2b_traffic_warm.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --rounds 2 --e2e-steps 2 > gpurun_out/r2b_ncu_warm.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke_ncu.log 2>&1
tail -3 gpurun_out/r2b_pytest.log; grep -h "ERROR SUMMARY\|rc=" gpurun_out/r2b_sanitize_*.log
