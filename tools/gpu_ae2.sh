# launch list of AE steps (tcgen05 passes) under ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ae2_launches.csv python tools/ae_bench.py --dims paper --steps 3 --warmup 1 > gpurun_out/ae2_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ae_(enc|dec|encw)_tc" -s 3 -c 3 -o gpurun_out/ae2_full python tools/ae_bench.py --dims paper --steps 2 --warmup 1 > gpurun_out/ae2_ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/ae2_*
