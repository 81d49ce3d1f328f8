python tools/kbench.py 8 2>&1 | head -1
SMOE_FUSED_NO_L2PF=1 python tools/kbench.py 8 2>&1 | head -1
SMOE_DOWN_L2=1 SMOE_SPLIT_FFN=1 python tools/kbench.py 8 2>&1 | head -1
python tools/phase_run.py on_demand 2>&1 | grep -E "ffn down phase" | grep -v " 0 0 0 0 0 0 0 0 | 0" | head -12
