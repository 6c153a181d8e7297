cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "multi_gpu" > gpurun_out/r2i_pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest2.log
for n in 1 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n tools/c5_run.py > gpurun_out/r2i_c5_n$n.json 2> gpurun_out/r2i_c5_n$n.err
  echo "n=$n rc=$?"
done
tail -3 gpurun_out/r2i_pytest2.log
for n in 1 2 4; do grep "^{" gpurun_out/r2i_c5_n$n.json | tail -1; tail -2 gpurun_out/r2i_c5_n$n.err; done
