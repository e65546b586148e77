"""TEST INFRASTRUCTURE: a CPU backend for paper_1309_1889_b200.parallel.

It runs the sharded parareal driver on CPU under gloo. The fine and coarse
propagations go through the oracle's propagate, which is the bitwise C
restatement of src/integrate.cpp:13-36 over msm_potential. The state algebra
follows the reference's exact operation order (src/parareal.cpp:58-90).
Sums are sequential: np.cumsum is sequential, unlike np.sum. This makes a
sharded run comparable bit for bit with the oracle's own parareal_run.

States are torch CPU tensors of shape (6, n), the layout of DeviceBackend.
Deltas are flat tensors: dpos (n Vec3s), dvel (n Vec3s), then rms_pos.
Never imported by the product path.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle_lib
from paper_1309_1889_b200 import _ERR, Error, ForceField, ParticleSystem


class OracleMsm(ForceField):
    """A stand-in ForceField carrying MSM parameters for the host backend."""

    def __init__(self, a, h, levels, kc=332.0636):
        self.a, self.h, self.levels, self.kc = a, h, levels, kc

    def name(self):
        return "msm"


def _seqsum(x):
    return float(np.cumsum(x)[-1]) if len(x) else 0.0


def _norm2(d):  # vec3.hpp:19-20: x*x + y*y + z*z, left to right
    return (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]


class HostBackend:
    device = None

    def __init__(self, cfg, v: ParticleSystem, kind: str = "port", fail=None):
        self.chk = oracle_lib.checker(kind)
        self.cfg = cfg
        self.v = v
        self.n = v.size()
        self.fail = fail or {}          # {fine-call number: (exception class, message)} for error tests
        self.fine_calls = 0

    def from_system(self, s):
        return torch.from_numpy(np.ascontiguousarray(np.concatenate([s.positions.T, s.velocities.T])))

    def to_host(self, st):
        a = st.numpy()
        return np.ascontiguousarray(a[:3].T), np.ascontiguousarray(a[3:].T)

    def empty_delta(self):
        return torch.empty(6 * self.n + 1, dtype=torch.float64)

    def propagate(self, which, st):
        sp = self.cfg.fine if which == "fine" else self.cfg.coarse
        if which == "fine":
            self.fine_calls += 1
            if self.fine_calls in self.fail:
                cls, msg = self.fail[self.fine_calls]
                raise cls(msg)
        ff = sp.force_field
        pos, vel = self.to_host(st)
        p, v, _, err = self.chk.propagate(pos, vel, self.v.charges, self.v.masses, self.v.box, ff.a, ff.h,
                                          ff.levels, sp.dt, sp.steps_per_slice, ff.kc,
                                          self.cfg.units.energy_to_native)
        if err is not None:
            raise _ERR.get(err.code, Error)(err.msg)
        return torch.from_numpy(np.ascontiguousarray(np.concatenate([p.T, v.T])))

    def sub(self, a, b):  # state_sub, src/parareal.cpp:58-73
        an, bn = a.numpy(), b.numpy()
        dpos = (an[:3] - bn[:3]).T
        dvel = (an[3:] - bn[3:]).T
        rms = np.sqrt(_seqsum(_norm2(dpos)) / (3.0 * self.n))
        return torch.from_numpy(np.concatenate([dpos.reshape(-1), dvel.reshape(-1), [rms]]))

    def add(self, base, d):  # state_add, src/parareal.cpp:75-82
        dn = d.numpy()
        dpos = dn[: 3 * self.n].reshape(-1, 3).T
        dvel = dn[3 * self.n: 6 * self.n].reshape(-1, 3).T
        out = base.numpy().copy()
        out[:3] += dpos
        out[3:] += dvel
        return torch.from_numpy(out)

    def rms_change(self, a, b):  # rms_pos_change, src/parareal.cpp:86-90
        d = (a.numpy()[:3] - b.numpy()[:3]).T
        return float(np.sqrt(_seqsum(_norm2(d)) / (3.0 * self.n)))

    @staticmethod
    def delta_rms(d):
        return float(d[-1])

    @staticmethod
    def clone(st):
        return st.clone()
