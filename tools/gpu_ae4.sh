cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "autoencoder or run_experiment" > gpurun_out/ae4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ae4_pytest.log
tail -n 15 gpurun_out/ae4_pytest.log
timeout 300 python tools/ae_bench.py --dims paper > gpurun_out/ae4_bench.json 2> gpurun_out/ae4_bench.err; echo "bench rc=$?"
cat gpurun_out/ae4_bench.json; tail -n 5 gpurun_out/ae4_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ae4_launches.csv python tools/ae_bench.py --dims paper --steps 2 --warmup 1 > gpurun_out/ae4_ncu.log 2>&1; echo "ncu rc=$?"
