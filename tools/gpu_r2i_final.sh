# final-code measurement set (round 2i): full GPU suite, smoke, bench 20 / 1000, reference arm,
# ncu launch list, DRAM traffic (cold / warm) of k_wide2 + k_post_small, ncu --set full of k_wide2 (launched)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i_pytest.log
tail -n 3 gpurun_out/r2i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2i_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench20.json 2> gpurun_out/r2i_bench20.err; echo "bench20 rc=$?"
timeout 900 python bench.py --steps 1000 --warmup 5 > gpurun_out/r2i_bench1000.json 2> gpurun_out/r2i_bench1000.err; echo "bench1000 rc=$?"
LTFB_STREAM_PROF=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ae > /dev/null 2> gpurun_out/r2i_stream_prof.txt; echo "prof rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2i_reference.json 2> gpurun_out/r2i_reference.err; echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ae > gpurun_out/r2i_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for cc in all none; do
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control $cc -k regex:'k_wide2|k_post_small' -s 30 -c 6 --csv --log-file gpurun_out/r2i_traffic_$cc.csv python bench.py --steps 40 --no-cpu-baseline --no-ae > gpurun_out/r2i_traffic_$cc.log 2>&1; echo "ncu traffic $cc rc=$?"
done
LTFB_NO_STREAM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide2 --launch-skip 4 -c 1 -o gpurun_out/r2i_wide2 python tools/step_driver.py --steps 8 > gpurun_out/r2i_ncu.log 2>&1; echo "ncu full rc=$?"
