"""Worker of tests/test_gpu_ipc_two_process.py: one rank of a two-process run on ONE GPU, collectives over a
gloo process group through the host-transport communicator (dho2g_comm_init_host), so the fused HVP ->
reduce-scatter exchanges CUDA-IPC handles and stores into the other process's receive buffer.

    python tests/ipc_worker.py RANK WORLD PORT OUT.npz ROUTE SMALL"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2505_00982_b200 as d  # noqa: E402
from oracle.bindings import blobs_dataset  # noqa: E402


def main():
    rank, world, port, out, route, small = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4],
                                           int(sys.argv[5]), int(sys.argv[6]))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def allgather(b):
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return b"".join(p.numpy().tobytes() for p in parts)

    ctx = d.Context(0)
    ctx.comm_init_host(rank, world, allgather)
    ctx.set_option("hvp_route", route)
    ctx.set_option("mlp_small", small)
    sizes = [20, 16, 12, 5]
    X, y = blobs_dataset(96, 20, 5, seed=3)
    mlp = d.MlpOracle(ctx, sizes)
    w = mlp.init_params(1)
    op = d.mlp_hvp_operator(ctx, mlp, w, d.Batch(X, y, 5))
    n = mlp.dim()
    st = d.lanczos_distributed(ctx, 12, op, n, 77)
    ops = [r[1] for r in ctx.ledger()]
    np.savez(out, diag=st.tridiag.diag, off=st.tridiag.offdiag, ops=np.array(ops),
             ipc=ctx.stat("nccl_calls"))
    st.close()
    op.close()
    mlp.close()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
