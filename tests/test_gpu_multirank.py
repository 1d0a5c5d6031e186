"""The multi-rank library path executed: 2 and 3 PROCESSES share this box's one GPU, each a rank of a
world > 1 krylov_project (no paper passage: the paper ran on one CPU).

NCCL needs one GPU per rank, so the ranks use the host transport (krylov_comm_create_host): every collective of
the library — the per-step scalar all-gather of the z-slab partition (PAR1), its halo exchange, the final
coefficient / statistics gather of the direction partition (PAR2) — is an all-gather of host buffers done by
torch.distributed over gloo. No kernel waits on another process (each collective synchronises its own stream on
the host). With the peer-memory transport on top (CUDA IPC, the step kernel stores the halo planes into the
neighbours' buffers), the host all-gather after every step orders those stores. Every rank's coefficients must
equal the oracle's (1e-9 floored), the world-1 run's, and each other's bitwise; verdicts identical."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import workloads as W
from tests.parity import assert_coeff

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def case(name):
    if name.startswith("zslab_bc"):  # the paper's heat model, adaptive k (Alg. 4) on z-slabs: large route + PAR1
        return W.heat_paper(16, k_max=400, n_steps=200), dict(part="zslab")
    if name.startswith("zslab"):
        return W.heat(24, 4, 25, n_steps=100, step=0.02, mz=26), dict(part="zslab")
    if name == "dirs_c1":
        return W.config1(), dict(part="dirs")
    if name == "dirs_c2s":
        return W.config2(n=2000, n_gen=5, n_steps=300, k=30), dict(part="dirs")
    if name == "dirs_heat":  # fused stencil Lanczos with several directions, sharded
        p = W.heat(20, 3, 20, n_steps=60, step=0.02)
        p["gens"] = [W.box((0, 0, 0), (3, 3, 3)), W.box((5, 6, 7), (9, 9, 9)), W.rand(3), W.box((19, 0, 0), (20, 20, 2))]
        p["z_lo"] = np.array([0.9, -1.0, 0.0, 0.5])
        p["z_hi"] = np.array([1.1, 1.0, 1.0, 1.5])
        return p, dict(part="dirs")
    raise KeyError(name)


def worker(rank, world, port, name, thresholds, q):
    import torch
    import torch.distributed as dist
    from paper_1804_01583_b200 import KrComm, KrylovReach, torch_allgather_bytes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = None
    try:
        torch.cuda.set_device(0)
        comm = KrComm.host(rank, world, 0)
        assert comm.selftest(reps=2), "host-transport all-gather self test"
        p, kw = case(name)
        with KrylovReach(p, device=0, comm=comm, **kw) as h:
            on = h.attach_peers(rank, world, torch_allgather_bytes, dist.barrier) if name.endswith("ipc") else False
            coeff, stats = h.project()
            cb = h.check_box(thresholds)
            again, _ = h.project()  # the same handle projects twice
            dist.barrier()          # nobody destroys (and frees IPC-mapped buffers) while a neighbour still runs
        q.put((rank, coeff, stats, cb, on, bool(np.array_equal(coeff, again)), None))
    except Exception as e:  # report, do not hang the other ranks
        q.put((rank, None, None, None, False, False, repr(e)))
    finally:
        if comm is not None:
            comm.close()
        dist.destroy_process_group()


def run_world(name, world, thresholds):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, name, thresholds, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
    assert all(r[6] is None for r in res), [r[6] for r in res]
    return res


@pytest.mark.parametrize("name,world", [("zslab", 2), ("zslab", 3), ("zslab_ipc", 2), ("zslab_ipc", 3),
                                        ("zslab_bc", 2), ("dirs_c1", 2), ("dirs_c1", 3), ("dirs_c2s", 2),
                                        ("dirs_heat", 3)])
def test_multirank_processes_on_one_gpu(name, world):
    from paper_1804_01583_b200 import KrylovReach
    from tests.test_gpu_parity import choose_property
    p, kw = case(name)
    adaptive = p.get("eps", 0.0) > 0.0
    ref = oracle.krylov_project_adaptive(p) if adaptive else oracle.krylov_project(p)
    thresholds = [choose_property(oracle.check_box(p, ref["coeff"], []))]
    with KrylovReach(p, device=0) as h:  # world 1
        c1, s1 = h.project()
        cb1 = h.check_box(thresholds)
    res = run_world(name, world, thresholds)
    for rank, coeff, stats, cb, on, same, _ in res:
        assert same, (name, rank, "second project differs")
        assert np.array_equal(coeff, res[0][1]), (name, rank, "ranks differ")
        assert_coeff(coeff, ref["coeff"], f"{name} world={world} rank={rank} vs oracle")
        assert_coeff(coeff, c1, f"{name} world={world} rank={rank} vs world 1")
        assert [s["k_eff"] for s in stats] == [s["k_eff"] for s in s1]
        assert (cb["found"], cb["step"], cb["row"]) == (cb1["found"], cb1["step"], cb1["row"])
        if name.endswith("ipc"):
            assert on, (name, rank, "peer-memory halo transport not enabled")
    if adaptive:
        assert [s["k_eff"] for s in res[0][2]] == [r["k_eff"] for r in ref["per_dir"]]


def test_nccl_one_rank_graph_capture():
    """NCCL itself on this one-GPU box: a 1-rank communicator from a broadcast unique id (the KrComm path of
    bench.py), its all-gather captured in a CUDA graph and replayed (krylov_comm_selftest — the same call the
    z-slab run makes every Krylov step), and a krylov_project on a handle that carries the communicator."""
    from paper_1804_01583_b200 import KrComm, KrylovReach
    comm = KrComm(0, 1, 0, lambda data: data)
    try:
        assert comm.selftest(reps=4)
        p = W.heat(20, 3, 12, n_steps=40)
        with KrylovReach(p, device=0, comm=comm, part="zslab") as h:
            coeff, _ = h.project()
        assert_coeff(coeff, oracle.krylov_project(p)["coeff"], "1-rank NCCL communicator")
    finally:
        comm.close()
