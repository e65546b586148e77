"""Extended-XYZ I/O against the reference's own load_system /
save_system / TrajectoryWriter (src/xyz_io.cpp), byte for byte and message for message.
CPU only."""
import ctypes as C

import numpy as np
import pytest

import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import xyz_io

_D = C.POINTER(C.c_double)


def _p(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_D)


def _sigs(ref):
    L = ref.lib
    L.ref_save_system.argtypes = [C.c_int64, _D, _D, _D, _D, _D, C.c_char_p, C.c_char_p, C.c_int]
    L.ref_load_system.argtypes = [C.c_char_p, C.c_int64, C.POINTER(C.c_int64), _D, _D, _D, _D, _D, C.c_char_p,
                                  C.c_int]
    L.ref_write_trajectory.argtypes = [C.c_int64, _D, _D, _D, _D, _D, C.c_int, C.c_char_p, C.c_char_p, C.c_int]
    for f in (L.ref_save_system, L.ref_load_system, L.ref_write_trajectory):
        f.restype = C.c_int


def ref_save(ref, s, path):
    _sigs(ref)
    buf = C.create_string_buffer(512)
    rc = ref.lib.ref_save_system(len(s.charges), _p(s.positions), _p(s.velocities), _p(s.charges), _p(s.masses),
                                 _p(s.box), str(path).encode(), buf, 512)
    assert rc == 0, buf.value


def ref_load(ref, path, cap=100000):
    _sigs(ref)
    n = C.c_int64()
    pos, vel, q, m, box = np.zeros((cap, 3)), np.zeros((cap, 3)), np.zeros(cap), np.zeros(cap), np.zeros(3)
    buf = C.create_string_buffer(512)
    rc = ref.lib.ref_load_system(str(path).encode(), cap, C.byref(n), pos.ctypes.data_as(_D), vel.ctypes.data_as(_D),
                                 q.ctypes.data_as(_D), m.ctypes.data_as(_D), box.ctypes.data_as(_D), buf, 512)
    if rc:
        return None, buf.value.decode()
    k = n.value
    return pkg.ParticleSystem(pos[:k], vel[:k], q[:k], m[:k], box), None


def systems():
    rng = np.random.default_rng(9)
    n = 257
    box = np.array([40.0, 17.25, 3.0e2])
    pos = rng.uniform(0, 1, (n, 3)) * box
    pos[0] = [0.0, 0.0, 0.0]
    pos[1] = box  # on the upper faces: inside (p <= box)
    vel = rng.normal(0, 1e-2, (n, 3))
    vel[2] = [-0.0, 1e-300, -3.5e-310]
    q = rng.choice([-0.834, 0.417, 1.0, -1.0], n)
    m = rng.choice([16.0, 1.008, 18.0], n)
    yield pkg.ParticleSystem(pos, vel, q, m, box)
    yield pkg.ParticleSystem(np.array([[1.0, 2.0, 3.0]]), np.zeros((1, 3)), np.array([0.1]), np.array([1e-3]),
                             np.array([1e5, 1e-5 + 3.0, 7.0]))


@pytest.mark.parametrize("k", [0, 1])
def test_save_load_byte_identical_to_reference(ref, tmp_path, k):
    s = list(systems())[k]
    a, b = tmp_path / "ours.xyz", tmp_path / "ref.xyz"
    xyz_io.save_system(s, str(a))
    ref_save(ref, s, b)
    assert a.read_bytes() == b.read_bytes()
    t = xyz_io.load_system(str(b))
    r, err = ref_load(ref, a)
    assert err is None
    for x, y in [(t.positions, s.positions), (t.velocities, s.velocities), (t.charges, s.charges),
                 (t.masses, s.masses), (t.box, s.box), (r.positions, t.positions), (r.masses, t.masses)]:
        assert np.array_equal(x, y)
        assert np.array_equal(np.signbit(x), np.signbit(y))  # -0.0 round-trips too


def test_trajectory_frames_byte_identical(ref, tmp_path):
    s = list(systems())[0]
    a, b = tmp_path / "ours_traj.xyz", tmp_path / "ref_traj.xyz"
    w = xyz_io.TrajectoryWriter(str(a))
    for f in range(3):
        w.write_frame(s, f * 10, f * 0.25)
    w.close()
    _sigs(ref)
    buf = C.create_string_buffer(512)
    assert ref.lib.ref_write_trajectory(len(s.charges), _p(s.positions), _p(s.velocities), _p(s.charges),
                                        _p(s.masses), _p(s.box), 3, str(b).encode(), buf, 512) == 0
    assert a.read_bytes() == b.read_bytes()


BAD = {
    "empty": "",
    "count_word": "abc\nbox 1 1 1\n",
    "count_zero": "0\nbox 1 1 1\n",
    "count_trailing": "2 x\nbox 1 1 1\n",
    "no_comment": "1\n",
    "no_box": "1\nfoo 1 1 1\nX 0 0 0 1 0 0 0 1\n",
    "box_short": "1\nbox 1 1\nX 0 0 0 1 0 0 0 1\n",
    "box_nan": "1\nbox 1 nan 1\nX 0 0 0 1 0 0 0 1\n",
    "row_fields": "2\nbox 5 5 5\nX 0 0 0 1 0 0 0 1\nX 1 1 1 1 0 0 0\n",
    "row_number": "1\nbox 5 5 5\nX 0 0 0 1e 0 0 0 1\n",
    "row_inf": "1\nbox 5 5 5\nX 0 0 inf 1 0 0 0 1\n",
    "eof": "3\nbox 5 5 5\nX 0 0 0 1 0 0 0 1\n",
    "mass": "2\nbox 5 5 5\nX 0 0 0 1 0 0 0 1\nX 1 1 1 1 0 0 0 0\n",
    "outside": "2\nbox 5 5 5\nX 0 0 0 1 0 0 0 1\nX 1 6 1 1 0 0 0 1\n",
    "crlf_ok": "1\r\nbox 5 5 5 step=3\r\nX 1 2 3 -1 0.5 0 0 2\r\n",
    "extra_tokens_ok": "1\nbox 5 5 5 anything goes here\nX 1 2 3 -1 0.5 0 0 2\n",
    "hexfloat_ok": "1\nbox 0x1p2 5 5\nX 1 2 3 -1 0.5 0 0 2\n",
}


@pytest.mark.parametrize("name", sorted(BAD))
def test_parse_errors_match_reference(ref, tmp_path, name):
    f = tmp_path / f"{name}.xyz"
    f.write_bytes(BAD[name].encode())
    r, err = ref_load(ref, f)
    try:
        s = xyz_io.load_system(str(f))
        ours = None
    except pkg.Error as e:
        ours = str(e)
    assert ours == err
    if err is None:
        assert np.array_equal(s.positions, r.positions) and np.array_equal(s.box, r.box)
