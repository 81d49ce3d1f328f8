export PYTHONFAULTHANDLER=1
mkdir -p gpurun_out/parity
PARITY_REPORT_DIR=gpurun_out/parity timeout 1200 python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider -s 2>&1 | grep -E "parity-fast|passed|failed|Error|error" | cut -c1-600
for md in exact fast; do echo "== $md"; SMOE_DECODE_MODE=$md timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-250; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_fast.py > gpurun_out/gputests3.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests3.txt
