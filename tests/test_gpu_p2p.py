"""The peer-memory halo transport's host protocol and memory path across PROCESSES (CUDA IPC export,
all-gather of the blobs, open, test-pattern stores into the neighbours' halo planes, verification, enable /
close), run as 2 and 3 processes on the one GPU of this box with gloo for the collectives — no kernel waits
on another process. The step kernel's halo stores themselves are the code path the virtual-slab tests run
(tests/test_gpu_parity.py, test_gpu_next1.py); a multi-GPU run adds only NVLink between the two."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import workloads as W
    from paper_1804_01583_b200 import KrylovReach, torch_allgather_bytes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        p = W.heat(20, 3, 8, n_steps=10, mz=6 + rank)  # per-rank slab heights differ (blob carries nz)
        with KrylovReach(p) as h:
            on = h.attach_peers(rank, world, torch_allgather_bytes, dist.barrier)
            # this world-1 handle must not run with the neighbours attached: close the mappings again,
            # and nobody frees its buffers before every rank has closed its mappings
            from paper_1804_01583_b200 import _abi as A
            A.check(A.lib().krylov_p2p_enable(h.h, 0))
            dist.barrier()
        dist.barrier()
        q.put((rank, on, getattr(h, "p2p_error", None)))
    except Exception as e:  # report, do not hang the other ranks
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_ipc_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(err is None for _, _, err in res), res
    assert all(on for _, on, _ in res), res
