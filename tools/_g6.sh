./tools/decision_bench
python -m pytest tests/test_gpu_offload_modes.py -q -x > gpurun_out/g6.log 2>&1; tail -3 gpurun_out/g6.log
python tools/ktrace_run.py 8 1.0 greedy > gpurun_out/ktrace_dec.txt 2>&1; grep -E "==|predictor|router" gpurun_out/ktrace_dec.txt | head -24
python tools/phase_run.py prefetch 2>&1 | grep -E "predictor \[" | head -8
