export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_prefill_tc.py -x -q -p no:cacheprovider 2>&1 | tail -2
SMOE_TC_NO_TMAP=1 timeout 600 python -m pytest tests/test_gpu_prefill_tc.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python tools/prefill_bench.py 48 512 1.0 batched,tensor 2>&1 | tail -3
timeout 600 python tools/prefill_bench.py 48 2048 1.0 batched,tensor 2>&1 | tail -3
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_tc_ffn" -c 4 -o gpurun_out/r02_ncu_tc3 -f python tools/prefill_bench.py 2 512 1.0 tensor > gpurun_out/ncu_tc.log 2>&1; echo "ncu full rc=$?"
