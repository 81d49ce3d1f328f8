python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity_scale.py tests/test_gpu_hybrid.py -q -x -k "batch or hybrid" 2>&1 | tail -3
python tools/batch_offload.py g20 8 0.25 > gpurun_out/batch_g20.txt 2>&1; tail -6 gpurun_out/batch_g20.txt
python tools/batch_offload.py mx 6 0.5 > gpurun_out/batch_mx.txt 2>&1; tail -7 gpurun_out/batch_mx.txt
