export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests2.txt 2>&1; rc=$?; echo "tests rc=$rc" >> gpurun_out/gputests2.txt
tail -4 gpurun_out/gputests2.txt
if [ $rc -ne 0 ]; then
  for f in tests/test_gpu*.py; do timeout 600 python -m pytest $f -m gpu -x -q -p no:cacheprovider > gpurun_out/t_$(basename $f .py).txt 2>&1; echo "$f rc=$?"; done
fi
timeout 300 python tools/phase_run.py on_demand > gpurun_out/phase_od.txt 2>&1
timeout 300 python tools/phase_run.py prefetch > gpurun_out/phase_pf.txt 2>&1
grep -h "ffn_gu\|ffn_down\|predictor\|true router" gpurun_out/phase_od.txt gpurun_out/phase_pf.txt | head -40
