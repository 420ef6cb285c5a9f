"""Experiment: two ranks sharing one GPU (torchrun --nproc-per-node 2), each fitting its row shard of
C2 through the sharded path with a 2-rank NCCL communicator; rank 0 compares the model with the
oracle's unsharded fit.  NCCL may refuse two ranks on one device; the script reports either way.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/two_rank_one_gpu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_2410_02425_b200 as lp  # noqa: E402
import synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(lp.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    uid = bytes(t.numpy().tobytes())
    torch.cuda.set_device(0)
    try:
        ctx = lp.Context(0, torch.cuda.current_stream(), uid, rank, world)
    except Exception as e:   # noqa: BLE001
        print("rank %d: communicator refused: %s" % (rank, e), flush=True)
        return 0
    full = synth.make_scaled(200)   # 25,600 rows
    sh = synth.make_scaled(200, rank, world)
    kw = dict(n_trees=6, max_depth=6)
    gm = lp.fit(ctx, sh.X, sh.y, lp.hparams(**kw), sh.users_col, sh.llm_id, sh.prof_id, sh.n_llm, sh.n_prof, 100.0,
                50.0, row_offset=sh.row_offset, n_global=sh.n_global)
    e = gm.export()
    if rank == 0:
        om = oracle.fit(full.X, full.y, oracle.hparams(**kw), full.users_col, full.llm_id, full.prof_id, full.n_llm,
                        full.n_prof, 100.0, 50.0)
        ok = (np.array_equal(om.feat, e["feat"]) and np.array_equal(om.val.view(np.uint32), e["val"].view(np.uint32))
              and np.array_equal(om.base.view(np.uint32), e["base"].view(np.uint32)))
        print("two ranks on one GPU, sharded fit vs unsharded oracle: %s" % ("BIT-EXACT" if ok else "MISMATCH"),
              flush=True)
    ctx.close()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
