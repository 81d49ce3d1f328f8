export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench2.json; tail -5 gpurun_out/bench2.err
