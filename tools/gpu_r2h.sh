cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2h_gpus.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k multi_gpu > gpurun_out/r2h_pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest2.log
for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 600 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_n$n.json 2> gpurun_out/r2h_bench_n$n.err
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_n$n.json 2> gpurun_out/r2h_bench_n$n.err; fi
done
tail -3 gpurun_out/r2h_pytest2.log
python -c "
import json
for n in (1,2,4):
    try:
        d=json.loads([l for l in open(f'gpurun_out/r2h_bench_n{n}.json').read().splitlines() if l.startswith('{')][-1]); print(n, d['value'], d['ms_per_step'], d['round_ms'], d['rounds_timed'], d['e2e']['value'])
    except Exception as e: print(n, 'failed', e)
"
