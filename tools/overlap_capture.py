"""Capture for the copy-overlap study (tools only; DESIGN.md §5 "Copy overlap").

    python tools/overlap_capture.py [steps]      # GPU: writes gpurun_out/overlap_trace.npz

Headline workload (Q30 shape, router-pf with 2000-token calibration, 32-token
prompt, teacher-forced random_token_stream(4)), experts resident (routing does
not depend on the cache): the executed and true ids of both offload modes and
router-pf predictions 1..4 layers ahead (smoe_predict_ahead) of the prefetch
run, plus the resident TPOTs and the link rate for the time model.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2603_19289_b200 import ModelConfig, Session
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    c = dict(bench.CONFIGS["q30"])
    L, K = c["layers"], c["top_k"]
    P = 32
    S = P + steps
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=S + 16)
    s.init_weights_seeded()
    s.preload_all()
    s.calibrate(2000, 2, 256)
    s.set_predictor("router-pf")
    s.set_decode_mode(os.environ.get("SMOE_DECODE_MODE", "fast"))
    prompt = bench.token_stream(P, c["vocab"], 3)
    forced = bench.token_stream(steps, c["vocab"], 4)
    out = {}
    for mode in ("on_demand", "prefetch"):
        s.reset(S, True)
        s.prefill(prompt)
        s.decode_stream(mode, forced)
        out[f"{mode}_true"] = s.trace("id_true", S).reshape(S, L, K)[P:]
        out[f"{mode}_exec"] = s.trace("id_exec", S).reshape(S, L, K)[P:]
        out[f"{mode}_resident_ms"] = np.array(s.token_ms())
        if mode == "prefetch":
            for d in (1, 2, 3, 4):
                out[f"ahead{d}"] = s.predict_ahead(0, S, d)[P:]
    out["link_GBps"] = np.array(s.measure_link(32))
    s.close()
    path = os.path.join(ROOT, "gpurun_out", "overlap_trace.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez(path, **out)
    print("saved", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
