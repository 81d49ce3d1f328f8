"""Expert-parallel combine decomposition on CPU with a real 2-process gloo group
(SURVEY §8e): experts are owned by rank e % world; each rank evaluates only its
experts' raw outputs for the executed decision and contributes them into a
zero-initialised [k][H] buffer; an all-reduce (sum) of that buffer is exact
because every row has exactly one non-zero contributor (x + 0 = x), so the
decision-order mixture every rank then computes equals moe_block bit for bit.
This is the arithmetic the GPU's peer-store combine (k_ffn_down / k_ep_mix)
relies on."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.bindings import Config

CFG = dict(layers=2, experts=8, top_k=3, hidden=32, expert_hidden=24, vocab=64, head_dim=8,
           seed=5)


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.bindings import Oracle
        orc = Oracle(threads=1)
        om = orc.build_model(Config(**CFG), round_bf16=True)
        t = om.generate_trace([1, 2, 3], 4, outputs=True)
        H, K, E = CFG["hidden"], CFG["top_k"], CFG["experts"]
        ok = True
        owned = [e for e in range(E) if e % world == rank]
        for s in range(t.ids.shape[0]):
            for l in range(CFG["layers"]):
                buf = torch.zeros(K, H, dtype=torch.float32)
                for i, e in enumerate(t.ids[s, l]):
                    if e % world != rank:
                        continue
                    wg = om.tensor(f"layer{l}.expert{e}.w_gate").reshape(CFG["expert_hidden"], H)
                    wu = om.tensor(f"layer{l}.expert{e}.w_up").reshape(CFG["expert_hidden"], H)
                    wd = om.tensor(f"layer{l}.expert{e}.w_down").reshape(H, CFG["expert_hidden"])
                    buf[i] = torch.from_numpy(orc.expert_ffn(wg, wu, wd, t.s[s, l]))
                dist.all_reduce(buf)  # exact: one contributor per row
                y = buf.numpy()
                out = np.zeros(H, np.float32)
                for i in range(K):  # decision order, f32 (model.cpp:297-301)
                    out = (out + np.float32(t.gates[s, l, i]) * y[i]).astype(np.float32)
                ok &= np.array_equal(y, t.outputs[s, l]) and np.array_equal(out, t.m[s, l])
        counts = torch.tensor([len(owned)])
        dist.all_reduce(counts)
        ok &= int(counts) == E
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_ep_combine_is_exact_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)], res
