export PYTHONFAULTHANDLER=1
mkdir -p gpurun_out/parity
PARITY_REPORT_DIR=gpurun_out/parity timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.json
