timeout 1500 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"
tail -3 gpurun_out/bench3.err
