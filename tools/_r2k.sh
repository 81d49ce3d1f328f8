export PYTHONFAULTHANDLER=1
for md in exact fast; do echo "== $md"; SMOE_DECODE_MODE=$md timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-250; done
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests4.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests4.txt
