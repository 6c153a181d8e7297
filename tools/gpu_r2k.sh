cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 1 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2977$n tools/c5_run.py > gpurun_out/r2k_c5_n$n.json 2> gpurun_out/r2k_c5_n$n.err
  echo "n=$n rc=$?"
done
for n in 1 2 4; do grep "^{" gpurun_out/r2k_c5_n$n.json | tail -1; tail -n 2 gpurun_out/r2k_c5_n$n.err | grep -v OMP; done
