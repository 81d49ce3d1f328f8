export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider 2>&1 | tail -2
SMOE_DECODE_MODE=fast timeout 200 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-400
SMOE_NO_FFN_CS_FUSED=1 SMOE_DECODE_MODE=fast timeout 200 python tools/kbench.py 16 2>&1 | tail -3 | head -2 | cut -c1-300
