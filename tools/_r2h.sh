export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider 2>&1 | tail -2
for md in exact fast; do echo "== $md"; SMOE_DECODE_MODE=$md timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-250; done
timeout 900 python tools/long_context.py 12 1024 16384 2>&1 | tail -3
