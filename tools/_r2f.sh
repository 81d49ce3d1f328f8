export PYTHONFAULTHANDLER=1
mkdir -p gpurun_out/parity
PARITY_REPORT_DIR=gpurun_out/parity timeout 1500 python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider -s 2>&1 | grep -E "parity-fast|passed|failed|Error|error" | cut -c1-300
timeout 900 python tools/long_context.py 16 1024 4096 2>&1 | tail -4
timeout 900 python tools/long_context.py 12 16384 2>&1 | tail -3
