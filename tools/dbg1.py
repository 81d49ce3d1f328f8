import sys, ctypes as C, numpy as np, time
sys.path.insert(0, ".")
from paper_2603_19289_b200 import ModelConfig, Session
cfg = dict(layers=3, experts=6, top_k=2, hidden=16, expert_hidden=24, vocab=32, head_dim=8, seed=11)
s = Session(ModelConfig(**cfg), cache_fraction=0.5, max_positions=64, deadlock_s=2.0)
s.init_weights_seeded()
def dbg():
    out = np.zeros(32, np.int32)
    s.lib.smoe_debug_state(s._h, out.ctypes.data_as(C.c_void_p), 32)
    print("dbg", list(out[:6 + 6]))
dbg()
s.reset(8, True)
try:
    s.prefill([1, 2])
except Exception as e:
    print("ERR", e)
dbg()
time.sleep(1)
dbg()
