# C5 rounds with the row-major eval mapping: parity subset, then C5 at N = 2 / 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "eval or tournament or run_experiment" > gpurun_out/c5e_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/c5e_pytest.log
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n tools/c5_run.py > gpurun_out/c5e_n$n.json 2> gpurun_out/c5e_n$n.err; echo "c5 n$n rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c5e_n$n.json').read().strip().splitlines()[-1]); print($n, d['samples_per_s'], d['ms_per_step'], d['rounds'])"
done
