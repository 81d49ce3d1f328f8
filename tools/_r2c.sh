for md in exact fast; do for w in 1 3; do echo "== $md W=$w"; SMOE_DECODE_MODE=$md SMOE_GU_WARPS=$w timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-250; done; done
