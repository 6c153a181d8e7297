# parity of the working tree + interleaved A/B (tools/ab/lib_*.so: base = HEAD, new = working tree, new2 = optional)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
[ -z "$AB_NOTEST" ] && timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/ab3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab3_pytest.log
tail -n 2 gpurun_out/ab3_pytest.log
V="base new"; [ -f tools/ab/lib_new2.so ] && V="base new new2"
for st in ${AB_STEPS:-200}; do for i in 1 2 3; do for v in $V; do
env ${AB_ENV_new2:+$( [ $v = new2 ] && echo $AB_ENV_new2 )} LTFB_LIB_PATH=$PWD/tools/ab/lib_$v.so timeout 300 python bench.py --steps $st --warmup 5 --no-cpu-baseline --no-ae 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); p=d['stream_profile_us']; print('$v s$st', round(d['ms_per_step']*1000,2), {k: round(v,2) for k,v in p.items()}, round(d['kernels_ms_per_launch']['wide']*1000,2))"
done; done; done
