# 4-GPU box: full GPU suite (incl. the 2-GPU tests), then bench at N = 1 / 2 / 4 as the driver launches it
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2i4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i4_pytest.log
tail -n 3 gpurun_out/r2i4_pytest.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2i4_n1.json 2> gpurun_out/r2i4_n1.err; echo "n1 rc=$?"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2i4_n$n.json 2> gpurun_out/r2i4_n$n.err; echo "n$n rc=$?"
done
for n in 1 2 4; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2i4_n$n.json') if l.startswith('{')][-1]); print($n, d['value'], d['ms_per_step'], d.get('round_ms'), d['e2e']['value'])"; done
