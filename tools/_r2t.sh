export PYTHONFAULTHANDLER=1
timeout 900 python tools/prefill_bench.py 48 512 1.0 batched,tensor 2>&1 | tail -4
timeout 900 python tools/prefill_bench.py 48 2048 1.0 batched,tensor 2>&1 | tail -4
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(pf_|tc_)" --csv --log-file gpurun_out/r02_prefill_tc_launches.csv python tools/prefill_bench.py 2 512 1.0 tensor > gpurun_out/ncu_pf.log 2>&1; echo "ncu launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_tc_(gu|down)" -c 4 -o gpurun_out/r02_ncu_tc -f python tools/prefill_bench.py 2 512 1.0 tensor > gpurun_out/ncu_tc.log 2>&1; echo "ncu full rc=$?"
