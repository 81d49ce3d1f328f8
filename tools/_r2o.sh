export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider -k "toy or L3 or L2" 2>&1 | tail -3
for md in fast exact; do echo "== $md"; SMOE_DECODE_MODE=$md timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-400; done
echo "== fast + L2 prefetch"; SMOE_L2_PREFETCH=1 SMOE_DECODE_MODE=fast timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-400
