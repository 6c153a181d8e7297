# 4 GPUs of one box: the multi-GPU parity tests, then bench at N = 1 / 2 / 4 (driver command, 20 steps; and 1,000 steps)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/n4_gpus.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/n4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/n4_pytest.log
for st in 20 1000; do
for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 600 python bench.py --steps $st --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/n4_bench_${st}_n$n.json 2> gpurun_out/n4_bench_${st}_n$n.err
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n --steps $st --warmup 5 --no-cpu-baseline --no-ae > gpurun_out/n4_bench_${st}_n$n.json 2> gpurun_out/n4_bench_${st}_n$n.err; fi
done; done
tail -3 gpurun_out/n4_pytest.log
python -c "
import json
for st in (20, 1000):
  for n in (1,2,4):
    try:
        d=json.loads([l for l in open(f'gpurun_out/n4_bench_{st}_n{n}.json').read().splitlines() if l.startswith('{')][-1]); print(st, n, d['value'], d['ms_per_step'], d['round_ms'], d['rounds_timed'], d['e2e']['value'])
    except Exception as e: print(st, n, 'failed', e)
"
