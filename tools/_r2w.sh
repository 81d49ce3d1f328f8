export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -p no:cacheprovider -k expert_parallel 2>&1 | grep -v "^$" | tail -40
