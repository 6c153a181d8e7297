cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in 16 0; do
LTFB_WIDE_V2=1 LTFB_W2_FLAGS=$f LTFB_STREAM_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ae > gpurun_out/w2g_$f.json 2> gpurun_out/w2g_$f.err; echo "flags=$f rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/w2g_$f.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels_ms_per_launch']['wide'], d['stream_profile_us'])"
grep -A 30 "stream prof" gpurun_out/w2g_$f.err | tail -10 | head -9
done
LTFB_WIDE_V2=1 LTFB_NO_STREAM=1 timeout 600 ncu --cache-control none --clock-control none -k regex:k_wide2 --launch-skip 4 -c 1 --metrics lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__bytes_read.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum python tools/step_driver.py --steps 8 > gpurun_out/w2g_ncu.log 2>&1; echo "ncu rc=$?"; grep -E "lts__|dram__|l1tex__|gpu__time" gpurun_out/w2g_ncu.log
