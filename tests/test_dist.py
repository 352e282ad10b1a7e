"""Multi-GPU path (include/gc_dist.h, paper_1606_06025_b200/dist.py).

CPU (gloo, world_size 2): the round driver and its two per-round all-gathers run over a real
torch.distributed gloo group; each rank's partition kernels are replaced by a numpy test
double with the kernels' per-phase semantics (FakePartition), so the host logic — partition
bounds, local CSR slices, packing, all-gather of variable-size pair lists, termination by
global |W| — is exercised exactly as on GPUs.  The gathered colouring must equal the oracle.

GPU: the real kernels, P partitions inside one process (exchange = in-process), must give
the single-GPU colouring bit for bit for P = 1..8 (partition invariance).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads as wl

COMMIT = 0x80000000
CMASK = 0x7FFFFFFF


class FakePartition:
    """numpy model of one gc_dist partition (test double for the CUDA kernels)."""

    def __init__(self, n_global, v_begin, v_end, rp_local, ci_local, policy="higher_id"):
        import torch
        self.torch = torch
        self.n, self.vb, self.ve = n_global, v_begin, v_end
        self.rp, self.ci = np.asarray(rp_local), np.asarray(ci_local)
        self.policy = policy
        self.st = np.ones(n_global, dtype=np.uint32)        # everyone pending with tent 1
        self.W = list(range(v_begin, v_end))
        self.Wn = []
        self.round = 1

    def adj(self, v):
        i = v - self.vb
        return self.ci[self.rp[i]:self.rp[i + 1]]

    def recolors(self, v, w):
        return v > w if self.policy == "higher_id" else v < w

    def phase_a(self):
        if self.round == 1:
            return
        for v in self.W:
            used = {int(self.st[w] & CMASK) for w in self.adj(v) if self.st[w] & COMMIT}
            c = 1
            while c in used:
                c += 1
            self.st[v] = c

    def phase_b(self):
        lose = []
        for v in self.W:
            t = self.st[v] & CMASK
            if any((self.st[w] & CMASK) == t and self.recolors(v, int(w)) for w in self.adj(v)):
                lose.append(v)
        ls = set(lose)
        for v in self.W:
            if v not in ls:
                self.st[v] |= COMMIT
        self.Wn = lose
        return len(lose)

    def pack(self, what):
        vs = [v for v in self.W if what == 0 or (self.st[v] & COMMIT)]
        out = np.zeros(2 * len(vs), dtype=np.uint32)
        out[0::2] = vs
        out[1::2] = self.st[vs] if vs else []
        return self.torch.from_numpy(out.view(np.int32).copy())

    def unpack(self, pairs):
        a = pairs.cpu().numpy().view(np.uint32)
        self.st[a[0::2]] = a[1::2]

    def next_round(self):
        self.W, self.Wn = self.Wn, []
        self.round += 1

    def finalize(self):
        c = self.st[self.vb:self.ve] & CMASK
        return self.torch.from_numpy(c.astype(np.int32)), int(c.max()) if len(c) else 0, self.round


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


GRAPHS = {"rmat": lambda: wl.rmat(10, 8, seed=3), "mesh": lambda: wl.mesh2d(24, 17, 0.3, seed=2),
          "k9": lambda: wl.complete(9), "path": lambda: wl.path(33)}


def _worker(rank, world, port, name, policy, q):
    import torch
    import torch.distributed as dist
    from paper_1606_06025_b200.dist import TorchComm, local_slice, run_rounds
    from paper_1606_06025_b200 import partition_edge_balanced
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        g = GRAPHS[name]()
        bounds = partition_edge_balanced(g.row_ptr, world)
        b, e = int(bounds[rank]), int(bounds[rank + 1])
        rpl, cil = local_slice(g.row_ptr, g.col_idx, b, e)
        part = FakePartition(g.n, b, e, rpl, cil, policy)
        res = run_rounds([part], TorchComm())
        q.put((rank, b, e, res.colors_local[0].numpy().tolist(), res.num_colors, res.rounds, res.exchanged_pairs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("policy", ["higher_id", "lower_id"])
def test_gloo_world2_matches_oracle(name, policy):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, policy, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort()
    g = GRAPHS[name]()
    colors = np.zeros(g.n, dtype=np.uint32)
    for rank, b, e, c, nc, r, sent in outs:
        colors[b:e] = c
    ref, nc_ref, r_ref = oracle.sgr(g, policy)
    assert np.array_equal(colors, ref)
    assert all(o[4] == nc_ref and o[5] == r_ref for o in outs)
    assert sum(o[6] for o in outs) > 0


def test_local_slice_and_bounds():
    from paper_1606_06025_b200.dist import local_slice
    from paper_1606_06025_b200 import partition_edge_balanced
    g = wl.rmat(9, 8)
    b = partition_edge_balanced(g.row_ptr, 3)
    rebuilt = []
    for k in range(3):
        rpl, cil = local_slice(g.row_ptr, g.col_idx, int(b[k]), int(b[k + 1]))
        assert rpl[0] == 0 and rpl[-1] == len(cil)
        rebuilt.append(cil)
    assert np.array_equal(np.concatenate(rebuilt), g.col_idx)


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("policy", ["higher_id", "lower_id"])
def test_gpu_partition_invariance(parts, policy):
    """P partitions on one GPU == single-GPU gc_color == oracle, bit for bit."""
    import torch
    import paper_1606_06025_b200 as gc
    from paper_1606_06025_b200.dist import color_partitioned
    for g in (wl.rmat(13, 8, seed=4), wl.mesh2d(64, 48, 0.3), wl.complete(40), wl.star(300, center_last=True)):
        rp = torch.from_numpy(g.row_ptr).cuda()
        ci = torch.from_numpy(g.col_idx if g.m else np.zeros(1, np.int32)).cuda()
        colors, nc, rounds = color_partitioned(rp, ci, parts, policy)
        one = gc.color(rp, ci, policy=policy)
        ref, nc_ref, r_ref = oracle.sgr(g, policy)
        assert torch.equal(colors.cpu(), one.colors.cpu())
        assert np.array_equal(colors.cpu().numpy().view(np.uint32), ref)
        assert nc == nc_ref == one.num_colors and rounds == r_ref == one.rounds


@pytest.mark.gpu
def test_gpu_dist_degree_policy_unsupported():
    import torch
    import paper_1606_06025_b200 as gc
    from paper_1606_06025_b200.dist import color_partitioned
    g = wl.path(10)
    with pytest.raises(gc.GcError):
        color_partitioned(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(), 2, "degree")
