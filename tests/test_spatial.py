"""Spatial decomposition: csrc/msmb_dd.cu + parallel.SpatialDecomposition.

CPU:
* the per-part work plans tile the pair columns and every level's planes exactly;
* the exchange is exact under gloo with world_size 2: it is an int64 MAX over
  IEEE bit patterns, with unowned entries set to INT64_MIN.

GPU (one device; the parts run in-process through the same phase/exchange
sequence that torchrun ranks run): a decomposed trajectory equals the
single-GPU one bit for bit, for several part counts and config shapes.
Errors surface identically.
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


SPECIAL = np.array([0.0, -0.0, 1.5, -2.25, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1.7976931348623157e308,
                    -1e-310, 3.0, -7.0, 2.0 ** -1074, -(2.0 ** 1023), 0.1])


def _xworker(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bits = torch.from_numpy(SPECIAL.view(np.int64).copy())
        own = torch.arange(len(SPECIAL)) % world == rank
        buf = torch.where(own, bits, torch.full_like(bits, torch.iinfo(torch.int64).min))
        # two local parts on this rank: the second owns nothing
        other = torch.full_like(bits, torch.iinfo(torch.int64).min)
        parallel.exchange_max_bits([buf, other])
        np.save(os.path.join(out, f"x{rank}.npy"), np.stack([buf.numpy(), other.numpy()]))
    finally:
        dist.destroy_process_group()


def test_exchange_is_bit_exact_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_xworker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        for r in range(2):
            got = np.load(os.path.join(d, f"x{r}.npy"))
            for row in got:
                assert np.array_equal(row, SPECIAL.view(np.int64))


# ------------------------------------------------------------------------------ GPU
def _single(w, steps):
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    ds = pkg.DeviceSystem(f, s)
    ds.propagate(w.dt, steps)
    return ds.download(), f


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,parts,steps", [("c2s", 30000, 1, 2), ("c2s", 30000, 2, 3), ("c2s", 30000, 3, 2), ("c5", 20000, 4, 2),
                                                ("c4", 30000, 3, 2), ("c1s", 2048, 7, 3)])
def test_decomposed_trajectory_bitwise(name, n, parts, steps):
    w = fx.config(name, n_override=n)
    if name == "c5":
        w.dt = 0.02  # short survivable slice of the fine propagator shape
    if name == "c4":
        w.dt = 0.02
    (pos1, vel1), f1 = _single(w, steps)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=parts)
    out, energy = dd.propagate(w.dt, steps)
    assert np.array_equal(out.positions, pos1)
    assert np.array_equal(out.velocities, vel1)
    ref = pkg.msm_potential(pkg.ParticleSystem(pos1, vel1, w.q, w.mass, w.box), pkg.MsmConfig(w.a, w.h, w.levels))
    assert abs(energy - ref.total_energy) <= 1e-12 * abs(ref.total_energy)


@pytest.mark.gpu
def test_decomposed_single_evaluation_energy():
    w = fx.config("c2s", n_override=30000)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=4)
    out, energy = dd.propagate(w.dt, 0)
    ref = pkg.msm_potential(s, pkg.MsmConfig(w.a, w.h, w.levels))
    assert np.array_equal(out.positions, w.pos) and abs(energy - ref.total_energy) <= 1e-12 * abs(ref.total_energy)


@pytest.mark.gpu
def test_decomposed_errors_match_single_gpu():
    w = fx.config("c1s", n_override=1024)
    pos = w.pos.copy()
    pos[300] = [1e3, 0.0, 0.0]  # outside grid coverage
    s = pkg.ParticleSystem(pos, w.vel, w.q, w.mass, w.box)
    with pytest.raises(pkg.CoverageError) as e1:
        pkg.propagate(pkg.PropagatorSpec(pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels)), w.dt, 2), s)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=3)
    with pytest.raises(pkg.CoverageError) as e2:
        dd.propagate(w.dt, 2)
    assert str(e1.value) == str(e2.value)
    p, v = dd.parts[0][1].download()
    assert np.array_equal(p, pos)  # state restored


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [2, 3])
def test_decomposed_rebuilds_and_calls_bitwise(parts):
    # a tiny skin makes the list (and so atom ownership) change mid-trajectory: the
    # velocities then travel from the old owners (lazy velocity exchange); two calls
    # reuse the list across the call boundary.  Bit-identical to one GPU run the same way.
    w = fx.config("c1s", n_override=2048)
    dt, skin = 0.05, 0.002
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    f.set_pair_skin(skin)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    ds = pkg.DeviceSystem(f, s)
    ds.propagate(dt, 12)
    ds.propagate(dt, 9)
    pos1, vel1 = ds.download()
    nreb = f.work_counters()["list_rebuilds"]
    assert nreb > 3
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, local_parts=parts)
    for fp, _, _ in dd.parts:
        fp.set_pair_skin(skin)
    dd.propagate(dt, 12, download=False)
    out, _ = dd.propagate(dt, 9)
    assert dd.parts[0][0].work_counters()["list_rebuilds"] == nreb
    assert np.array_equal(out.positions, pos1)
    assert np.array_equal(out.velocities, vel1)
