python tools/kbench.py 8 > gpurun_out/kbench_fused.txt 2>&1; cat gpurun_out/kbench_fused.txt
SMOE_SPLIT_FFN=1 python tools/kbench.py 8 > gpurun_out/kbench_split.txt 2>&1; cat gpurun_out/kbench_split.txt
python tools/ktrace_run.py 8 1.0 greedy > gpurun_out/ktrace_fused.txt 2>&1; head -60 gpurun_out/ktrace_fused.txt
SMOE_SPLIT_FFN=1 python tools/ktrace_run.py 8 1.0 greedy > gpurun_out/ktrace_split.txt 2>&1; grep "==" gpurun_out/ktrace_split.txt
python -m pytest tests -m gpu -x -q > gpurun_out/g4_tests.log 2>&1; tail -5 gpurun_out/g4_tests.log
