# C5 at 1 / 2 / 4 GPUs on the final code (10 M desk samples sharded over the ranks' HBM stores)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29521 tools/c5_run.py > gpurun_out/r2i_c5_n1.json 2> gpurun_out/r2i_c5_n1.err; echo "c5 n1 rc=$?"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n tools/c5_run.py > gpurun_out/r2i_c5_n$n.json 2> gpurun_out/r2i_c5_n$n.err; echo "c5 n$n rc=$?"
done
for n in 1 2 4; do tail -c 600 gpurun_out/r2i_c5_n$n.json; echo; done
