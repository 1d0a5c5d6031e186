"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the z-slab partition
(krylov_zslab_range), the halo schedule (krylov_zslab_halo_plan — the same plan the NCCL transport and
the virtual-slab transport execute), the per-step all-gather of rank partial sums, and the NCCL
unique-id broadcast helper. The slab arithmetic is a numpy emulation of the fused lookahead step
(DESIGN §6), written independently of the CUDA code; with the library's partition and halo plan it
must reproduce the unpartitioned oracle Lanczos (Alg. 3)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W

M, MZ, BLK, K = 10, 13, 3, 12


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def stencil_w(ui, uim1, a, b, c, cx, cy, cz, zmask):
    """w on buffer planes 1..nz+1 from u_i (planes 0..nz+2) and u_{i-1} (planes 1..nz+1)."""
    core = ui[1:-1]
    up, dn = ui[2:], ui[:-2]
    pad = np.pad(core, ((0, 0), (1, 1), (1, 1)))
    sx = pad[:, 1:-1, :-2] + pad[:, 1:-1, 2:]
    sy = pad[:, :-2, 1:-1] + pad[:, 2:, 1:-1]
    Au = cx * sx + cy * sy + cz * (up + dn) - 2 * (cx + cy + cz) * core
    w = a * Au - b * core - c * uim1[1:-1]
    w[~zmask] = 0.0
    return w


def slab_partials(w, zoff, nz, cx, cy, cz, outs):
    """sum w^2, -w^T A w (edge form with Dirichlet ghosts), C w over owned planes (w planes 0..nz)."""
    own, above = w[:nz], w[1:nz + 1]
    wx = np.pad(own, ((0, 0), (0, 0), (0, 1)))[:, :, 1:]
    wy = np.pad(own, ((0, 0), (0, 1), (0, 0)))[:, 1:, :]
    D = cx * (wx - own) ** 2 + cy * (wy - own) ** 2 + cz * (above - own) ** 2
    D[:, :, 0] += cx * own[:, :, 0] ** 2
    D[:, 0, :] += cy * own[:, 0, :] ** 2
    if zoff == 0:
        D[0] += cz * own[0] ** 2
    vals = [np.sum(own ** 2), np.sum(D)]
    for o in outs:
        if o["kind"] == "all":
            vals.append(o["value"] * np.sum(own))
        else:
            (x0, y0, z0), (x1, y1, z1) = o["lo"], o["hi"]
            zs = slice(max(z0 - zoff, 0), max(min(z1 - zoff, nz), 0))
            vals.append(o["value"] * np.sum(own[zs, y0:y1, x0:x1]))
    return np.array(vals)


def slab_lanczos(rank, world, exchange, allgather):
    """Lookahead Lanczos on this rank's slab; returns (alpha[1..k], beta[1..k], P)."""
    from paper_1804_01583_b200 import krylov_zslab_halo_plan, krylov_zslab_range
    p = W.heat(M, BLK, K, mz=MZ)
    z0, z1 = krylov_zslab_range(MZ, world, rank)
    nz = z1 - z0
    plan = krylov_zslab_halo_plan(MZ, world, rank)
    cx = cy = 0.01 * (M + 1) ** 2
    cz = 0.01 * (MZ + 1) ** 2
    gen = W.dense_vec(p["gens"][0], p).reshape(MZ, M, M)
    u = [np.zeros((nz + 3, M, M)) for _ in range(3)]
    for bp in range(nz + 3):  # u_1 analytic on owned + halo planes
        gz = z0 - 1 + bp
        if 0 <= gz < MZ:
            u[0][bp] = gen[gz]
    zmask = np.array([z0 + q < MZ for q in range(nz + 1)])[:, None, None] & np.ones((1, M, M), bool)
    outs = p["outs"]
    red = allgather(slab_partials(u[0][1:nz + 2], z0, nz, cx, cy, cz, outs))
    b0 = np.sqrt(red[0])
    s = {1: 1 / b0}
    alpha = {1: -red[1] / red[0]}
    beta = {}
    P = [s[1] * red[2:]]
    for i in range(1, K + 1):
        cur, prev, nxt = (i - 1) % 3, (i - 2) % 3, i % 3
        c = beta[i - 1] * s[i - 1] if i > 1 else 0.0
        w = stencil_w(u[cur], u[prev], s[i], alpha[i] * s[i], c, cx, cy, cz, zmask)
        red = allgather(slab_partials(w, z0, nz, cx, cy, cz, outs))
        beta[i] = np.sqrt(red[0])
        if i == K:
            break
        s[i + 1] = 1 / beta[i]
        alpha[i + 1] = -red[1] / red[0]
        P.append(s[i + 1] * red[2:])
        u[nxt][1:nz + 1] = w[:nz]
        exchange(u[nxt], plan)
    return np.array([alpha[i] for i in range(1, K + 1)]), np.array([beta[i] for i in range(1, K + 1)]), \
        np.array(P).T


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1804_01583_b200 import torch_broadcast_id
        idb = torch_broadcast_id(bytes(range(128)) if rank == 0 else None)
        assert idb == bytes(range(128))

        def allgather(vec):
            t = torch.from_numpy(np.ascontiguousarray(vec))
            parts = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            tot = np.zeros_like(vec)
            for pr in parts:  # rank order, as lz_finalize sums the gathered rank vectors
                tot = tot + pr.numpy()
            return tot

        def exchange(buf, plan):
            reqs, recvs = [], []
            for is_send, peer, plane, n in plan:
                t = torch.from_numpy(np.ascontiguousarray(buf[plane:plane + n])) if is_send else \
                    torch.zeros((n,) + buf.shape[1:], dtype=torch.float64)
                reqs.append(dist.isend(t, peer) if is_send else dist.irecv(t, peer))
                if not is_send:
                    recvs.append((plane, n, t))
            for r in reqs:
                r.wait()
            for plane, n, t in recvs:
                buf[plane:plane + n] = t.numpy()

        a, b, P = slab_lanczos(rank, world, exchange, allgather)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), a=a, b=b, P=P)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_zslab_lanczos_gloo_matches_oracle(world, tmp_path):
    mp.spawn(_worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    p = W.heat(M, BLK, K, mz=MZ)
    ref = oracle.lanczos(p, oracle.directions(p)[0], K)
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for r in res[1:]:  # every rank computes bit-identical scalars
        assert np.array_equal(r["a"], res[0]["a"]) and np.array_equal(r["b"], res[0]["b"])
    assert np.allclose(res[0]["a"], ref["alpha"], rtol=1e-12, atol=0)
    assert np.allclose(res[0]["b"], ref["beta"], rtol=1e-12, atol=0)
    scale = np.abs(ref["P"]).max()
    assert np.max(np.abs(res[0]["P"] - ref["P"])) <= 1e-12 * scale


def test_single_rank_emulation_matches_oracle():
    """World size 1 (no halos): the emulation itself against Alg. 3."""
    a, b, P = slab_lanczos(0, 1, lambda buf, plan: None, lambda v: v)
    p = W.heat(M, BLK, K, mz=MZ)
    ref = oracle.lanczos(p, oracle.directions(p)[0], K)
    assert np.allclose(a, ref["alpha"], rtol=1e-12) and np.allclose(b, ref["beta"], rtol=1e-12)


def test_halo_plan_pairs_up():
    """Every receive is matched by the peer's send of the same size, and the received planes are the
    peer's owned planes adjacent to my slab (global plane bookkeeping)."""
    from paper_1804_01583_b200 import krylov_zslab_halo_plan, krylov_zslab_range
    for mz, world in [(13, 2), (13, 3), (1000, 8), (400, 8), (9, 4)]:
        for r in range(world):
            z0, z1 = krylov_zslab_range(mz, world, r)
            for is_send, peer, plane, n in krylov_zslab_halo_plan(mz, world, r):
                if is_send:
                    continue
                pz0, pz1 = krylov_zslab_range(mz, world, peer)
                match = [op for op in krylov_zslab_halo_plan(mz, world, peer) if op[0] and op[1] == r]
                assert len(match) == 1 and match[0][3] == n
                send_first_global = pz0 - 1 + match[0][2]  # peer buffer plane -> global z
                recv_first_global = z0 - 1 + plane
                assert send_first_global == recv_first_global
                assert pz0 <= send_first_global and send_first_global + n <= pz1  # peer's owned planes


def _par2_worker(rank, world, port, n_dir, out_dir):
    """Direction sharding (PAR2) host logic on gloo: each rank takes its directions from the library's
    partitioner (krylov_dirs_of_rank), fills its local coefficient block [(N+1)][o][ndl_max] with values that
    encode (step, row, global direction), and all-gathers the blocks in rank order — the exchange the library
    does with one collective after the Krylov loop; the gathered blocks are then reordered as the header states
    (local block dl of rank w is global direction w + dl * world)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1804_01583_b200 import krylov_dirs_of_rank
        mine = krylov_dirs_of_rank(n_dir, world, rank)
        ndl_max = -(-n_dir // world)
        np1, o = 7, 3
        loc = np.full((np1, o, ndl_max), np.nan)
        for dl, d in enumerate(mine):
            loc[:, :, dl] = 1000.0 * d + 10.0 * np.arange(o)[None, :] + 0.01 * np.arange(np1)[:, None]
        t = torch.from_numpy(loc)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        lists = [None] * world
        dist.all_gather_object(lists, mine)
        np.savez(os.path.join(out_dir, f"p{rank}.npz"), G=np.stack([q.numpy() for q in parts]),
                 lists=np.array([len(x) for x in lists]), flat=np.concatenate([np.array(x, dtype=np.int64) for x in lists]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_dir", [(2, 21), (3, 8), (3, 2), (2, 1)])
def test_direction_sharding_gloo(world, n_dir, tmp_path):
    mp.spawn(_par2_worker, args=(world, free_port(), n_dir, str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "p0.npz")
    flat = r0["flat"]
    assert sorted(flat.tolist()) == list(range(n_dir))  # a partition: every direction exactly once
    assert r0["lists"].tolist() == [len(range(w, n_dir, world)) for w in range(world)]
    G = r0["G"]  # [world][N+1][o][ndl_max]
    np1, o = G.shape[1], G.shape[2]
    coeff = np.empty((np1, o, n_dir))
    for d in range(n_dir):
        coeff[:, :, d] = G[d % world, :, :, d // world]
    want = 1000.0 * np.arange(n_dir)[None, None, :] + 10.0 * np.arange(o)[None, :, None] + \
        0.01 * np.arange(np1)[:, None, None]
    assert np.array_equal(coeff, want)
    for r in range(1, world):  # every rank gathered the same blocks
        assert np.array_equal(np.load(tmp_path / f"p{r}.npz")["G"], G, equal_nan=True)
