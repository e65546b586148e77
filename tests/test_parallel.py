"""Sharded parareal (paper_1309_1889_b200/parallel.py).

CPU tests: the shipped driver runs under gloo with world_size 1 and 2 on the
oracle-backed host backend (tests/parallel_host.py). Its trajectory must equal
the oracle's own parareal_run bit for bit, whatever the rank count. This
covers the skip heuristic, multiple windows and error agreement across ranks.

GPU tests: the device backend with one rank reproduces the single-GPU C++
driver (msmb_parareal_run) bit for bit; two processes sharing the one B200,
talking over gloo (CUDA tensors staged through the host: no kernel waits on
another process), reproduce it bit for bit as well; and the C++ driver's own
executor over fine-field replicas (GpuExecutor -> msmb_parareal_run_ex) equals
the single-field run, with the reference's report rows.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import rel_rms
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
from paper_1309_1889_b200 import parallel

FINE, COARSE = (8.0, 2.0, 2, 0.005, 8), (6.0, 3.0, 2, 0.02, 2)


def _system(n=256, seed=5):
    box = np.array([14.0, 14.0, 14.0])
    pos, q = fx.uniform(n, box, "random_neutral", 1.5, seed)
    mass = np.full(n, 18.0)
    vel = fx.maxwell_boltzmann(mass, 300.0, seed + 1)
    return pkg.ParticleSystem(pos, vel, q, mass, box)


def _host_cfg(window=3, max_iter=4, tol=1e-7, skip=1e-9):
    from parallel_host import OracleMsm
    fa, fh, fl, fdt, fs = FINE
    ga, gh, gl, gdt, gs = COARSE
    return pkg.PararealConfig(window, max_iter, tol, pkg.PropagatorSpec(OracleMsm(fa, fh, fl), fdt, fs),
                              pkg.PropagatorSpec(OracleMsm(ga, gh, gl), gdt, gs), skip_threshold=skip)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, total, cfg_kw, fail):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch.distributed as dist
    from parallel_host import HostBackend
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v = _system()
        cfg = _host_cfg(**cfg_kw)
        be = HostBackend(cfg, v, fail=(fail or {}).get(rank))
        try:
            res = parallel.parareal_run(v, total, cfg, backend=be)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"),
                     pos=np.stack([t.positions for t in res.trajectory]),
                     vel=np.stack([t.velocities for t in res.trajectory]),
                     counts=np.array([res.counts["g_evals"], res.counts["f_evals"], res.counts["f_skipped"],
                                      res.windows]),
                     fine_run=res.shard.fine_slices_run, rows=np.array([r[4] for r in res.report_rows]))
        except pkg.Error as e:
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), err_type=type(e).__name__, err_msg=str(e))
    finally:
        dist.destroy_process_group()


def _run_world(world, total=7, cfg_kw=None, fail=None):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), d, total, cfg_kw or {}, fail), nprocs=world,
                           join=True, start_method="spawn")
        return [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]


def _oracle(port, total=7, window=3, max_iter=4, tol=1e-7, skip=1e-9):
    v = _system()
    return port.parareal_run(v.positions, v.velocities, v.charges, v.masses, v.box, FINE, COARSE, window,
                             max_iter, tol, total, skip_threshold=skip)


def test_single_process_equals_oracle(port):
    from parallel_host import HostBackend
    v = _system()
    cfg = _host_cfg()
    res = parallel.parareal_run(v, 7, cfg, backend=HostBackend(cfg, v))
    tp, tv, cnt, err = _oracle(port)
    assert err is None and res.converged
    assert np.array_equal(np.stack([t.positions for t in res.trajectory]), tp)
    assert np.array_equal(np.stack([t.velocities for t in res.trajectory]), tv)
    assert [res.counts["g_evals"], res.counts["f_evals"], res.counts["f_skipped"], res.windows] == list(cnt[:4])
    assert res.shard.world == 1 and res.shard.fine_slices_run == res.counts["f_evals"]


def test_two_ranks_gloo_equal_oracle_bitwise(port):
    out = _run_world(2)
    tp, tv, cnt, err = _oracle(port)
    assert err is None
    for r in out:  # every rank holds the same, reference-exact trajectory
        assert np.array_equal(r["pos"], tp) and np.array_equal(r["vel"], tv)
        assert list(r["counts"]) == list(cnt[:4])
    # the fine sweep was split: ranks ran disjoint shares of f_evals
    runs = [int(r["fine_run"]) for r in out]
    assert sum(runs) == int(cnt[1]) and min(runs) >= 1


def test_two_ranks_window_and_no_skip(port):
    # window of 4 over 6 points, no skip heuristic, fixed iteration count (no short circuit)
    kw = dict(window=4, max_iter=2, tol=1e-3, skip=None)
    out = _run_world(2, total=6, cfg_kw=kw)
    tp, tv, cnt, err = _oracle(port, total=6, window=4, max_iter=2, tol=1e-3, skip=-1.0)
    assert err is None
    for r in out:
        assert np.array_equal(r["pos"], tp) and list(r["counts"]) == list(cnt[:4])


def test_error_agreement_across_ranks():
    # rank 1 fails on its first fine slice (slice 2), rank 0 on its second (slice 3):
    # every rank raises the lowest slice's error, as a sequential executor would
    fail = {1: {1: (pkg.CoverageError, "particle 17 outside grid coverage")},
            0: {2: (pkg.CoincidentParticlesError, "particles 1 and 2 coincide")}}
    out = _run_world(2, fail=fail)
    for r in out:
        assert str(r["err_type"]) == "CoverageError"
        assert str(r["err_msg"]) == "particle 17 outside grid coverage"


def test_validation_messages():
    v = _system(8)
    cfg = _host_cfg()
    cfg.coarse.steps_per_slice = 3
    with pytest.raises(pkg.ConfigError, match="span different slice lengths"):
        parallel.parareal_run(v, 2, cfg, backend=object())
    with pytest.raises(pkg.ConfigError, match="total_points must be >= 1"):
        parallel.parareal_run(v, 0, _host_cfg(), backend=object())


@pytest.mark.gpu
def test_device_backend_equals_cpp_driver_bitwise(port):
    v = _system()
    F = pkg.MsmField(pkg.MsmConfig(*FINE[:3]))
    G = pkg.MsmField(pkg.MsmConfig(*COARSE[:3]))
    cfg = pkg.PararealConfig(3, 4, 1e-7, pkg.PropagatorSpec(F, FINE[3], FINE[4]),
                             pkg.PropagatorSpec(G, COARSE[3], COARSE[4]), skip_threshold=1e-9)
    a = pkg.parareal_run(v, 7, cfg)
    b = parallel.parareal_run(v, 7, cfg)
    pa = np.stack([t.positions for t in a.trajectory])
    assert np.array_equal(pa, np.stack([t.positions for t in b.trajectory]))
    assert np.array_equal(np.stack([t.velocities for t in a.trajectory]),
                          np.stack([t.velocities for t in b.trajectory]))
    assert a.counts == b.counts and a.windows == b.windows
    tp, _, cnt, err = _oracle(port)
    assert err is None and rel_rms(pa, tp) <= 1e-8


def _gpu_worker(rank, world, port, out_dir):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        v = _system()
        F = pkg.MsmField(pkg.MsmConfig(*FINE[:3]))
        G = pkg.MsmField(pkg.MsmConfig(*COARSE[:3]))
        cfg = pkg.PararealConfig(3, 4, 1e-7, pkg.PropagatorSpec(F, FINE[3], FINE[4]),
                                 pkg.PropagatorSpec(G, COARSE[3], COARSE[4]), skip_threshold=1e-9)
        res = parallel.parareal_run(v, 7, cfg)
        np.savez(os.path.join(out_dir, f"g{rank}.npz"), pos=np.stack([t.positions for t in res.trajectory]),
                 vel=np.stack([t.velocities for t in res.trajectory]), fine_run=res.shard.fine_slices_run,
                 counts=np.array([res.counts["g_evals"], res.counts["f_evals"], res.counts["f_skipped"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_processes_device_backend_gloo_bitwise():
    v = _system()
    F = pkg.MsmField(pkg.MsmConfig(*FINE[:3]))
    G = pkg.MsmField(pkg.MsmConfig(*COARSE[:3]))
    cfg = pkg.PararealConfig(3, 4, 1e-7, pkg.PropagatorSpec(F, FINE[3], FINE[4]),
                             pkg.PropagatorSpec(G, COARSE[3], COARSE[4]), skip_threshold=1e-9)
    a = pkg.parareal_run(v, 7, cfg)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_gpu_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        out = [dict(np.load(os.path.join(d, f"g{r}.npz"))) for r in range(2)]
    pa = np.stack([t.positions for t in a.trajectory])
    va = np.stack([t.velocities for t in a.trajectory])
    for r in out:
        assert np.array_equal(r["pos"], pa) and np.array_equal(r["vel"], va)
        assert list(r["counts"]) == [a.counts["g_evals"], a.counts["f_evals"], a.counts["f_skipped"]]
    runs = [int(r["fine_run"]) for r in out]
    assert sum(runs) == a.counts["f_evals"] and min(runs) >= 1


@pytest.mark.gpu
def test_gpu_executor_replicas_bitwise(port):
    v = _system()
    F = pkg.MsmField(pkg.MsmConfig(*FINE[:3]))
    G = pkg.MsmField(pkg.MsmConfig(*COARSE[:3]))
    cfg = pkg.PararealConfig(3, 4, 1e-7, pkg.PropagatorSpec(F, FINE[3], FINE[4]),
                             pkg.PropagatorSpec(G, COARSE[3], COARSE[4]), skip_threshold=1e-9)
    a = pkg.parareal_run(v, 7, cfg)
    reps = [pkg.MsmField(pkg.MsmConfig(*FINE[:3])) for _ in range(2)]  # one per GPU; here all on cuda:0
    b = pkg.parareal_run(v, 7, cfg, exec=pkg.GpuExecutor(reps))
    assert np.array_equal(np.stack([t.positions for t in a.trajectory]), np.stack([t.positions for t in b.trajectory]))
    assert a.counts == b.counts and a.report_rows == b.report_rows and a.point_iterations == b.point_iterations
    assert len(b.report_rows) > 0 and len(b.point_iterations) == 7
    # against the reference's report (the driver over the oracle, bitwise the reference's
    # parareal_run on this fixture): same rows, converged flags and point iterations
    from parallel_host import HostBackend
    hcfg = _host_cfg()
    h = parallel.parareal_run(v, 7, hcfg, backend=HostBackend(hcfg, v))
    assert [r[:3] for r in b.report_rows] == [r[:3] for r in h.report_rows]
    assert [r[4] for r in b.report_rows] == [r[4] for r in h.report_rows]
    assert b.point_iterations == list(h.point_iterations)
