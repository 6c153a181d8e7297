cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "autoencoder or run_experiment" > gpurun_out/ae5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ae5_pytest.log
tail -n 15 gpurun_out/ae5_pytest.log
LTFB_AE_TIMING=1 timeout 300 python tools/ae_bench.py --dims paper --steps 20 --warmup 3 2>&1 | grep ae_timing | tail -3
timeout 300 python tools/ae_bench.py --dims paper; timeout 300 python tools/ae_bench.py --dims desk
