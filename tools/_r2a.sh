set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.txt
tail -30 gpurun_out/gputests.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
