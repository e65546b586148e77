"""Spatial slab decomposition: csrc/msmb_slab.cu +
parallel.SpatialDecomposition.

CPU:
* the per-part work plans tile the pair columns and every level's planes exactly;
* the torch.distributed plumbing of the NCCL bootstrap (the 128-byte unique id
  broadcast from rank 0) under gloo with world_size 2.

GPU (one device; the parts run in one process through the same plans, kernels and
exchange lists as torchrun ranks, with copies for the ncclSend/Recv): a decomposed
trajectory equals the single-GPU one (direct lattice method) bit for bit, for
several part counts and config shapes, including pair-list rebuilds with atom
migration between parts.  Errors surface identically.  The exchanged bytes per
step stay those of halos, not of whole buffers.
"""
import ctypes as C
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import _native, fixtures as fx
from paper_1309_1889_b200 import parallel

PLAN_CASES = [
    ((12.0, 2.5, 6), (144.0, 144.0, 144.0), 300000),   # C2
    ((12.0, 2.5, 4), (551.0, 551.0, 551.0), 1 << 24),  # C3
    ((12.0, 2.5, 5), (300.0, 650.0, 650.0), 12675000),  # C4 slab
    ((10.0, 2.5, 2), (40.0, 40.0, 40.0), 8192),        # C1
    ((8.0, 2.0, 2), (5.0, 5.0, 5.0), 16),              # tiny
]


def _plan(cfg, box, n, nparts, part):
    lib = _native.lib()
    c = pkg.MsmConfig(*cfg)._c()
    u = pkg.UnitsConfig.physical()._c()
    out = np.zeros(4 + 3 * 16, dtype=np.int32)
    rc = lib.msmb_dd_plan(C.byref(c), C.byref(u), np.asarray(box, dtype=np.float64).ctypes.data_as(C.POINTER(C.c_double)),
                          n, nparts, part, out.ctypes.data_as(C.POINTER(C.c_int32)), len(out))
    assert rc == 0
    ncx, cx0, cx1, levels = out[:4]
    planes = [tuple(out[4 + 3 * k: 7 + 3 * k]) for k in range(levels)]
    return ncx, (cx0, cx1), planes


@pytest.mark.parametrize("cfg,box,n", PLAN_CASES)
@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 7, 8])
def test_plans_tile_the_work(cfg, box, n, nparts):
    plans = [_plan(cfg, box, n, nparts, p) for p in range(nparts)]
    ncx = plans[0][0]
    cols = [p[1] for p in plans]
    assert cols[0][0] == 0 and cols[-1][1] == ncx
    for a, b in zip(cols, cols[1:]):
        assert a[1] == b[0] and a[0] <= a[1]
    for k in range(len(plans[0][2])):
        d0 = plans[0][2][k][0]
        rng = [(p[2][k][1], p[2][k][2]) for p in plans]
        assert rng[0][0] == 0 and rng[-1][1] == d0
        for a, b in zip(rng, rng[1:]):
            assert a[1] == b[0] and a[0] <= a[1]
        assert all(r[0] % 4 == 0 for r in rng)  # k_lattice tiles are 4 planes high


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _idworker(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # SpatialDecomposition's bootstrap: rank 0's id bytes reach every rank unchanged
        idbuf = bytes(range(128)) if rank == 0 else bytes(128)
        obj = [idbuf]
        dist.broadcast_object_list(obj, src=0)
        np.save(os.path.join(out, f"id{rank}.npy"), np.frombuffer(obj[0], dtype=np.uint8))
    finally:
        dist.destroy_process_group()


def test_nccl_id_broadcast_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_idworker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        for r in range(2):
            assert np.array_equal(np.load(os.path.join(d, f"id{r}.npy")), np.arange(128, dtype=np.uint8))


# ------------------------------------------------------------------------------ GPU
def _single(w, steps, dt=None, skin=None, calls=1, direct=True):
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    f.set_lattice_method(direct=direct)  # several parts: the direct stencil on owned planes
    if skin is not None:
        f.set_pair_skin(skin)
    ds = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    for _ in range(calls):
        ds.propagate(dt or w.dt, steps)
    return ds.download(), f


def _slab(w, parts, skin=None):
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=parts)
    if skin is not None:
        for f in dd.fields:
            f.set_pair_skin(skin)
    return dd


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,parts,steps", [("c2s", 30000, 1, 2), ("c2s", 30000, 2, 3), ("c2s", 30000, 3, 2),
                                                ("c5", 20000, 4, 2), ("c4", 30000, 3, 2), ("c1s", 2048, 2, 3)])
def test_decomposed_trajectory_bitwise(name, n, parts, steps):
    w = fx.config(name, n_override=n)
    if name in ("c5", "c4"):
        w.dt = 0.02  # short survivable slices of these shapes
    (pos1, vel1), f1 = _single(w, steps, direct=parts > 1)  # one part keeps the FFT lattice
    dd = _slab(w, parts)
    out, energy = dd.propagate(w.dt, steps)
    assert np.array_equal(out.positions, pos1)
    assert np.array_equal(out.velocities, vel1)
    ref = pkg.msm_potential(pkg.ParticleSystem(pos1, vel1, w.q, w.mass, w.box), pkg.MsmConfig(w.a, w.h, w.levels))
    assert abs(energy - ref.total_energy) <= 1e-10 * abs(ref.total_energy)
    st = dd.stats()
    assert st["parts"] == parts and (parts == 1 or st["halo"] > 0)


@pytest.mark.gpu
def test_nccl_transport_one_rank():
    """The NCCL transport (runtime-loaded libnccl, communicator init, all-reduce of the
    rebuild decision, all-gathers of counts, errors, energies and the final state) on a
    one-rank communicator: bitwise the local transport's result."""
    w = fx.config("c1s", n_override=4096)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    cfg = pkg.MsmConfig(w.a, w.h, w.levels)
    a, ea = parallel.SpatialDecomposition(cfg, s, local_parts=1).propagate(w.dt, 3)
    dn = parallel.SpatialDecomposition(cfg, s, transport="nccl")
    b, eb = dn.propagate(w.dt, 3)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.velocities, b.velocities)
    assert ea == eb
    with pytest.raises(pkg.CoverageError):  # errors through the NCCL all-gather of records
        bad = w.pos.copy()
        bad[11] = [1e3, 0.0, 0.0]
        parallel.SpatialDecomposition(cfg, pkg.ParticleSystem(bad, w.vel, w.q, w.mass, w.box),
                                      transport="nccl").propagate(w.dt, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [2, 3, 5])
def test_decomposed_migration_bitwise(parts):
    """Fast atoms and a tiny skin: the list is rebuilt every step and atoms migrate
    between parts; still bit-identical to one GPU."""
    w = fx.config("c1s", n_override=8192)
    rng = np.random.default_rng(5)
    w.vel = rng.normal(0.0, 0.05, size=w.vel.shape)  # A/fs: ~0.1 A per step at dt 2 fs
    dt, skin, steps = 2.0, 0.01, 4
    (pos1, vel1), f1 = _single(w, steps, dt=dt, skin=skin)
    dd = _slab(w, parts, skin=skin)
    out, _ = dd.propagate(dt, steps)
    st = dd.stats()
    assert st["rebuilds"] >= steps and st["migrated"] > 0
    assert np.array_equal(out.positions, pos1)
    assert np.array_equal(out.velocities, vel1)


@pytest.mark.gpu
def test_decomposed_errors_match_single_gpu():
    w = fx.config("c1s", n_override=4096)
    pos = w.pos.copy()
    pos[300] = [1e3, 0.0, 0.0]  # outside grid coverage
    s = pkg.ParticleSystem(pos, w.vel, w.q, w.mass, w.box)
    with pytest.raises(pkg.CoverageError) as e1:
        pkg.propagate(pkg.PropagatorSpec(pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels)), w.dt, 2), s)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=3)
    with pytest.raises(pkg.CoverageError) as e2:
        dd.propagate(w.dt, 2)
    assert str(e1.value) == str(e2.value) and e1.value.step == e2.value.step


@pytest.mark.gpu
def test_literal_abort_decomposed():
    """P1 under the decomposition: the literal C1 input aborts at the reference's step
    with the reference's particle."""
    w = fx.config("c1")
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    with pytest.raises(pkg.Error) as e1:
        pkg.propagate(pkg.PropagatorSpec(pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels)), w.dt, 5), s)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=2)
    with pytest.raises(pkg.Error) as e2:
        dd.propagate(w.dt, 5)
    assert type(e1.value) is type(e2.value) and str(e1.value) == str(e2.value)
    assert e1.value.step == e2.value.step


@pytest.mark.gpu
def test_halo_traffic_is_small():
    """Per step a part receives halo positions and lattice planes, far less than the
    whole-buffer exchanges of a replicated decomposition (~40 MB/step at C3 x 8)."""
    w = fx.config("c2s", n_override=120000)
    dd = _slab(w, 4)
    dd.propagate(w.dt, 2)
    st = dd.stats()
    whole = 8 * (6 * w.n) + 8 * sum(int(np.prod(d)) for d in pkg.grid_geometry(
        pkg.MsmConfig(w.a, w.h, w.levels), w.box)[0])
    assert 0 < st["bytes_per_step"] < 0.5 * whole
