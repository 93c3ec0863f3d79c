"""One rank of the horizon-sharded LQ solve (NEXT-2), for tests/test_gpu_horizon.py: torchrun with
gloo (ranks may share one GPU); rank 0 saves the assembled global solution."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_07823_b200 as P  # noqa: E402
from paper_2506_07823_b200 import horizon  # noqa: E402
from workloads import synth  # noqa: E402


def main():
    out_path, N, n, m, B, kind = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    qp = synth.random_lq(B, N, n, m, seed=77, kind=kind)
    qpt = {k: torch.from_numpy(v).cuda() for k, v in qp.items()}
    s, e = horizon.split_stages(N, world)[rank]
    loc = horizon.local_problem(qpt, s, e)
    h = P.PdIlqr(N=e - s - 1, n=n, m=m, batch=B, dtype=torch.float64)
    out = horizon.solve_lq_sharded(h, loc, qpt["P_term"], qpt["p_term"], qpt["dx0"], rank, world,
                                   horizon.dist_all_gather(dist, device=torch.device("cpu")))
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, {k: out[k].cpu().numpy() for k in ("dx", "du", "dlam", "info")})
    if rank == 0:
        dx = np.concatenate([p["dx"][:, :-1] for p in parts] + [parts[-1]["dx"][:, -1:]], axis=1)
        dl = np.concatenate([p["dlam"][:, :-1] for p in parts] + [parts[-1]["dlam"][:, -1:]], axis=1)
        du = np.concatenate([p["du"] for p in parts], axis=1)
        np.savez(out_path, dx=dx, du=du, dlam=dl, info=np.stack([p["info"] for p in parts]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
