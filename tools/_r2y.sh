ulimit -a | head -20; nproc; cat /sys/fs/cgroup/pids.max 2>/dev/null; cat /sys/fs/cgroup/pids/pids.max 2>/dev/null
timeout 600 python -X faulthandler -c "
import numpy as np, bench
from oracle.bindings import Config, Oracle
c=dict(bench.CONFIGS['q30']); c['layers']=4
om=Oracle().build_model(Config(**c), round_bf16=True)
print('built', flush=True)
d=om.calibrate(32,2,256)
print('calibrated', np.array(d.d).shape, flush=True)
" 2>&1 | tail -8
timeout 900 python -X faulthandler bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 800 gpurun_out/bench_ref.json; tail -5 gpurun_out/bench_ref.err
