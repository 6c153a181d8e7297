# clean 20-step bench (driver's command) x2, then DRAM traffic of k_wide2 / k_post_small cold and warm (r02g)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/m_bench20_$i.json 2> gpurun_out/m_bench20_$i.err; echo "bench20 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/m_bench20_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['stream_profile_us']['step_us'])"
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control all -k regex:'k_wide2|k_post_small' -s 30 -c 6 --csv python bench.py --steps 40 --no-cpu-baseline --no-ae > gpurun_out/m_traffic_cold.csv 2> gpurun_out/m_traffic_cold.err; echo "cold rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none -k regex:'k_wide2|k_post_small' -s 30 -c 6 --csv python bench.py --steps 40 --no-cpu-baseline --no-ae > gpurun_out/m_traffic_warm.csv 2> gpurun_out/m_traffic_warm.err; echo "warm rc=$?"
grep -E "dram__bytes|gpu__time" gpurun_out/m_traffic_cold.csv | head -12
