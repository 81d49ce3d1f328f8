export PYTHONFAULTHANDLER=1
echo "== default"; SMOE_DECODE_MODE=fast timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-330
for v in cc64s2 cc64s3 w8cc64s2; do echo "== $v"; SMOE_LIB=tools/variant/$v/libsmoe_b200.so SMOE_DECODE_MODE=fast timeout 300 python tools/kbench.py 16 2>&1 | tail -3 | cut -c1-330; done
