#!/bin/bash
# The GPU evidence of a round, run on one B200 through gpurun:
#   gpurun --timeout 3600 -- 'bash tools/gpu_round.sh [quick]'
# smoke, the GPU suite (parity reports under gpurun_out/parity), the bench
# line, the reference arm, and (unless `quick`) the ncu launch list of the
# bench command plus a full ncu capture of the tolerance-mode decode kernels.
# Everything lands in gpurun_out/; summaries go to profiles/ by hand
# (tools/launch_summary.py, tools/ncu_summary.py).
export PYTHONFAULTHANDLER=1
mkdir -p gpurun_out/parity
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
PARITY_REPORT_DIR=gpurun_out/parity timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
    > gpurun_out/gputests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests.txt
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref.json \
    2> gpurun_out/bench_ref.err; echo "reference arm rc=$?"
[ "$1" = "quick" ] && exit 0
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/launches.csv python bench.py --ncu --steps 4 --warmup 1 --calib-tokens 4 \
    --prompt-len 8 > gpurun_out/ncu_bench.log 2>&1; echo "ncu launch list rc=$?"
SMOE_DECODE_MODE=fast timeout 900 $NCU --set full --clock-control none --import-source on \
    --profile-from-start off -k regex:"k_(qkv|attn_fast|wo|router|ffn_gu_cs|ffn_down|final)" -c 14 \
    -o gpurun_out/ncu_fast -f python tools/ncu_target.py 8 4 --resident --profile-range \
    > gpurun_out/ncu_fast.log 2>&1; echo "ncu full rc=$?"
