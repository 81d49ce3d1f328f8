set -x
python -m pytest tests/test_gpu_offload_modes.py tests/test_gpu.py -x -q -k "offload or split_attention or kernel_limits or copy_lane or timeline or errors" > gpurun_out/g1_tests.log 2>&1; tail -5 gpurun_out/g1_tests.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck.txt 2>&1; tail -5 gpurun_out/san_memcheck.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_smoke.log
