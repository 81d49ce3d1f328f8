export PARITY_REPORT_DIR=gpurun_out/parity
python -m pytest tests/test_gpu_offload_modes.py tests/test_gpu_parity_scale.py -q -s -x --durations=0 > gpurun_out/g2_tests.log 2>&1; tail -25 gpurun_out/g2_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_smoke.log
