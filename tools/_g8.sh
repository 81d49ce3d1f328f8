python -m pytest tests/test_gpu_dropin.py -q -x 2>&1 | tail -3
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/$tool.txt 2>&1; echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|smoke ok' gpurun_out/san/$tool.txt | tr '\n' ' ')"
done
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_ffn_gu|k_ffn_down|k_router" -c 9 -o gpurun_out/ncu_offload python tools/ncu_target.py 4 4 --profile-range > gpurun_out/ncu_offload.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_offload.log
