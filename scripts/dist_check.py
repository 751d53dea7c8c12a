"""Multi-process partitioned solve check (torchrun): every rank runs its part
with NCCL boundary exchange; rank 0 compares the residual series with a
single-process solve bit-for-bit.  Usage:
  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/dist_check.py [case] [iters] [same_device]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2110_06879_b200 as ga  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "data/case118.m"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    same_device = len(sys.argv) > 3 and sys.argv[3] == "1"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = 0 if same_device else int(os.environ.get("LOCAL_RANK", rank))
    obj = [ga.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    net = ga.Network(case)
    cfg = ga.Config("case118", device=dev)
    sess = ga.Session.distributed(net, cfg, rank, world, obj[0])
    rec, _ = sess.iterate(iters)
    recs = [None] * world
    dist.all_gather_object(recs, rec.tolist())
    if rank == 0:
        ref = ga.Session(net, ga.Config("case118", device=dev))
        r1, _ = ref.iterate(iters)
        ok = all(np.array_equal(np.array(r).view(np.uint64)[:, :3], r1.view(np.uint64)[:, :3])
                 for r in recs)
        print(f"dist world={world} same_device={same_device} iters={len(rec)} bit_identical={ok}",
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
