"""Debug: NEXT-F4 NVLS setup + one verify at TP = 2 on tiny-tp (prints each step, hard timeouts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.multiprocessing as mp


def worker(rank, tp, nid, q):
    try:
        os.environ["SPECEDGE_TP_F4"] = "nvls"
        os.environ["SPECEDGE_DEBUG"] = "1"
        torch.cuda.set_device(rank)
        from paper_2505_17052_b200 import api
        from synth.configs import ModelShape
        from synth.trees import pooled_tree
        shape = ModelShape("tiny-tp", 2, 1024, 8, 8, 128, 2048, 1024, 1e-6, 10000.0)
        print(f"[{rank}] create", flush=True)
        m = api.Model(shape, 7, device=rank, max_position=1024, tp_rank=rank, tp_size=tp, nccl_id=nid)
        print(f"[{rank}] enable", flush=True)
        m.tp_fused_enable(4 * 65)
        print(f"[{rank}] mode {m.tp_fused_mode()}", flush=True)
        pool = api.KVPool(m, 16, 4)
        h = pool.alloc(300)
        pool.fill_random(h, 99, 1, 0)
        rng = np.random.default_rng(1)
        tr = pooled_tree(rng, 16, 4, 3, shape.vocab)
        ws = m.workspace(1, 17, 300)
        b = api.Batch.from_host([h], [100], [5], [1], [0], [tr], max_context_len=300)
        print(f"[{rank}] verify", flush=True)
        out = api.verify(m, pool, b, ws, auto_commit=False)
        torch.cuda.synchronize()
        print(f"[{rank}] done {out.row_target.cpu().numpy()[:8]}", flush=True)
        q.put((rank, "ok"))
    except Exception as e:
        import traceback
        q.put((rank, traceback.format_exc()))


if __name__ == "__main__":
    from paper_2505_17052_b200 import api
    nid = api.tp_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, nid, q)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in range(2):
        print(q.get(timeout=150), flush=True)
    for p in ps:
        p.join(timeout=30)
