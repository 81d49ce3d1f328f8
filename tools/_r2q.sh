export PYTHONFAULTHANDLER=1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.txt
NCU=/usr/local/cuda/bin/ncu
SMOE_DECODE_MODE=fast timeout 900 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_(qkv|attn_fast|wo|router|ffn_gu_cs|ffn_down|final)" -c 14 -o gpurun_out/r02_ncu_fast2 -f python tools/ncu_target.py 8 4 --resident --profile-range > gpurun_out/ncu_fast.log 2>&1; echo "ncu rc=$?"
for pol in lru lfu; do timeout 1500 python bench.py --cache-policy $pol --long-prompts 0 > gpurun_out/bench_$pol.json 2> gpurun_out/bench_$pol.err; echo "bench $pol rc=$?"; done
