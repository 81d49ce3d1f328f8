export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_prefill_tc.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/prefill_bench.py 48 512 1.0 batched,tensor 2>&1 | tail -3
timeout 900 python tools/prefill_bench.py 48 2048 1.0 batched,tensor 2>&1 | tail -3
for cap in 256 17000; do echo "== cap $cap"; KB_CAP=$cap SMOE_DECODE_MODE=fast timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | head -2 | cut -c1-300; KB_CAP=$cap SMOE_LIB=tools/variant/idlewait/libsmoe_b200.so SMOE_DECODE_MODE=fast timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | head -2 | cut -c1-300; done
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_tc_(gu|down)" -c 4 -o gpurun_out/r02_ncu_tc2 -f python tools/prefill_bench.py 2 512 1.0 tensor > gpurun_out/ncu_tc.log 2>&1; echo "ncu full rc=$?"
