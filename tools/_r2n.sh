export PYTHONFAULTHANDLER=1
timeout 900 python tools/overlap_capture.py 256 2>&1 | tail -2
NCU=/usr/local/cuda/bin/ncu
SMOE_DECODE_MODE=fast timeout 900 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_(qkv|attn|attn_fast|wo|router|ffn_gu|ffn_gu_w|ffn_down|final)" -c 14 -o gpurun_out/r02_ncu_fast -f python tools/ncu_target.py 8 4 --resident --profile-range > gpurun_out/ncu_fast.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_fast.log
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/r02_launches.csv python bench.py --ncu --steps 4 --warmup 1 --calib-tokens 4 --prompt-len 8 > gpurun_out/ncu_bench.log 2>&1; echo "ncu2 rc=$?"; tail -2 gpurun_out/ncu_bench.log
