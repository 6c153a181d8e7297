# AE tcgen05 column passes: parity tests, then timing vs the SIMT passes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "autoencoder" > gpurun_out/ae1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ae1_pytest.log
tail -n 30 gpurun_out/ae1_pytest.log
timeout 300 python tools/ae_bench.py --dims paper > gpurun_out/ae1_bench.json 2> gpurun_out/ae1_bench.err; echo "bench rc=$?"
cat gpurun_out/ae1_bench.json; tail -n 5 gpurun_out/ae1_bench.err
