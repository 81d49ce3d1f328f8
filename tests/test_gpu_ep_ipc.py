"""Expert parallelism across processes (one process per GPU in production):
two ranks exchange CUDA IPC handles over a gloo group and connect their peer
exchange buffers.  Both ranks share the one visible GPU here (IPC works across
processes on one device), so this exercises the multi-process path end to end
and checks bit-exact parity with the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOY = dict(layers=4, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32,
           seed=4)


def _rank(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.bindings import Config, Oracle
        from paper_2603_19289_b200 import ModelConfig, Session
        torch.cuda.set_device(0)
        orc = Oracle(threads=2)
        om = orc.build_model(Config(**TOY), round_bf16=True)
        table = om.calibrate(32, 2, 32)
        forced = np.array([(13 * i + 7) % TOY["vocab"] for i in range(6)], np.int32)
        want = om.generate_trace([1, 2, 3], 7, orc.make_predictor("router-pf", om, table),
                                 forced=forced)
        s = Session(ModelConfig(**TOY), cache_fraction=0.5, max_positions=64, ep_rank=rank,
                    ep_world=world)
        s.init_weights_seeded()
        s.load_default_vectors(np.array(table.d))
        s.set_predictor("router-pf")
        handles = [None] * world
        dist.all_gather_object(handles, s.ep_ipc_handles())
        s.ep_connect_ipc(handles)
        dist.barrier()
        S = 3 + 6
        s.reset(S, True)
        s.prefill([1, 2, 3])
        s.decode_stream("prefetch", forced)
        bad = [name for name, got, w in (("tokens", s.tokens(S)[2:], want.tokens),
                                         ("m", s.trace("m", S), want.m),
                                         ("logits", s.trace("logits", S), want.final_logits))
               if not np.array_equal(got, w)]
        ok = True if not bad else f"mismatch {bad}: tokens {s.tokens(S).tolist()} want {want.tokens.tolist()}"
        dist.barrier()
        s.close()
        q.put((rank, ok))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_ep_two_processes_ipc_bit_exact():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)], res
