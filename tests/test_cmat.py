"""CPU: CMAT file I/O through libadmm_b200.so (cmat_io.hpp), no GPU needed.

Restates the reference's Catch2 cases "cmat round trip is bit exact" and "cmat rejects
malformed files" (tests/test_problem_gen.cpp:105-164), adds the complex64 (CMF1)
variant, and — where oracle/_ref is built — runs every file through the unmodified
reference's read_cmat / read_cvec (oracle/ref_driver.cpp `cmat`) to pin the error
class, the FormatError byte offset and the payload bits against the reference itself.
The committed tests/golden/ref_gen_4x6_k2_seed3_{h,g}.cmat were written by the
reference's write_cmat (`admmsplit_ref gen out=DIR m=4 n=6 k=2 snr=inf seed=3 kind=cg`).
"""
import os
import subprocess

import numpy as np
import pytest

import paper_1811_05571_b200 as admm

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "admmsplit_ref")
GOLD = os.path.join(HERE, "golden")


def rand_c(rows, cols, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal((rows, cols)) + 1j * r.standard_normal((rows, cols))


def fnv(a: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    for b in np.ascontiguousarray(a, dtype=np.complex128).tobytes():
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def ref_read(path, vec=False):
    if not os.path.exists(REF):
        return None
    out = subprocess.run([REF, "cmat", f"in={path}", f"vec={int(vec)}"], capture_output=True, text=True,
                         check=True).stdout.split()
    return out


def ours(path, vec=False):
    try:
        a = admm.read_cvec(path) if vec else admm.read_cmat(path)
    except admm.FormatError as e:
        return ["error", "FormatError", str(e.byte_offset())], None
    except admm.IoError:
        return ["error", "IoError", "0"], None
    a2 = a.reshape(-1, 1) if vec else a
    return ["ok", str(a2.shape[0]), str(a2.shape[1]), fnv(a2)], a


def agree(path, vec=False):
    mine, arr = ours(path, vec)
    ref = ref_read(path, vec)
    if ref is not None:
        assert mine == ref[:len(mine)], (path, mine, ref)
    return mine, arr


def test_reference_written_files_read_bit_exact():
    p = admm.gen_problem(4, 6, 2, float("inf"), 3)
    h = admm.read_cmat(os.path.join(GOLD, "ref_gen_4x6_k2_seed3_h.cmat"))
    g = admm.read_cvec(os.path.join(GOLD, "ref_gen_4x6_k2_seed3_g.cmat"))
    assert h.dtype == np.complex128 and np.array_equal(h, p.h) and np.array_equal(g, p.g)
    assert admm.cmat_info(os.path.join(GOLD, "ref_gen_4x6_k2_seed3_h.cmat")) == (4, 6, "c128")


def test_round_trip_bit_exact(tmp_path):  # test_problem_gen.cpp:105-115
    a = rand_c(7, 5, 33)
    admm.write_cmat(tmp_path / "roundtrip.cmat", a)
    assert np.array_equal(admm.read_cmat(tmp_path / "roundtrip.cmat"), a)
    assert agree(tmp_path / "roundtrip.cmat")[0][3] == fnv(a)
    v = rand_c(9, 1, 34).reshape(-1)
    admm.write_cvec(tmp_path / "roundtrip_vec.cmat", v)
    assert np.array_equal(admm.read_cvec(tmp_path / "roundtrip_vec.cmat"), v)
    agree(tmp_path / "roundtrip_vec.cmat", vec=True)
    # byte layout is the reference's: header + interleaved little-endian binary64
    raw = (tmp_path / "roundtrip.cmat").read_bytes()
    assert raw[:4] == b"CMX1" and np.frombuffer(raw[4:20], "<u8").tolist() == [7, 5]
    assert raw[20:] == a.astype("<c16").tobytes()


def test_complex64_variant(tmp_path):
    a = rand_c(6, 10, 40)
    admm.write_cmat(tmp_path / "a64.cmat", a, dtype="c64")
    raw = (tmp_path / "a64.cmat").read_bytes()
    assert raw[:4] == b"CMF1" and len(raw) == 20 + 60 * 8
    assert admm.cmat_info(tmp_path / "a64.cmat") == (6, 10, "c64")
    r64 = admm.read_cmat(tmp_path / "a64.cmat", dtype="c64")
    assert r64.dtype == np.complex64 and np.array_equal(r64, a.astype(np.complex64))
    # widening read is exact
    assert np.array_equal(admm.read_cmat(tmp_path / "a64.cmat"), a.astype(np.complex64).astype(np.complex128))
    # an FP64 reference file read straight into complex64 storage rounds once
    admm.write_cmat(tmp_path / "a128.cmat", a)
    assert np.array_equal(admm.read_cmat(tmp_path / "a128.cmat", dtype="c64"), a.astype(np.complex64))
    # complex64 source written as CMX1 widens exactly
    admm.write_cmat(tmp_path / "w.cmat", a.astype(np.complex64))
    assert np.array_equal(admm.read_cmat(tmp_path / "w.cmat"), a.astype(np.complex64).astype(np.complex128))
    # the reference reads only CMX1: a CMF1 file is a bad magic there (offset 0)
    ref = ref_read(tmp_path / "a64.cmat")
    if ref is not None:
        assert ref == ["error", "FormatError", "0"]


def test_rejects_malformed_files(tmp_path):  # test_problem_gen.cpp:117-164
    empty = tmp_path / "empty.cmat"
    empty.write_bytes(b"")
    assert agree(empty)[0] == ["error", "FormatError", "0"]

    bad = tmp_path / "bad_magic.cmat"
    bad.write_bytes(b"NOPE" + bytes(16))
    assert agree(bad)[0] == ["error", "FormatError", "0"]

    trunc = tmp_path / "truncated.cmat"
    admm.write_cmat(trunc, rand_c(4, 4, 35))
    os.truncate(trunc, 20 + 3 * 16)
    assert agree(trunc)[0] == ["error", "FormatError", str(20 + 3 * 16)]

    trail = tmp_path / "trailing.cmat"
    admm.write_cmat(trail, rand_c(2, 2, 36))
    with open(trail, "ab") as f:
        f.write(b"x")
    assert agree(trail)[0] == ["error", "FormatError", str(20 + 4 * 16)]

    notvec = tmp_path / "not_vec.cmat"
    admm.write_cmat(notvec, rand_c(3, 2, 37))
    assert agree(notvec, vec=True)[0] == ["error", "FormatError", "12"]

    assert agree(tmp_path / "does_not_exist.cmat")[0] == ["error", "IoError", "0"]
    with pytest.raises(admm.ParameterError):
        admm.write_cvec(tmp_path / "empty_vec.cmat", np.zeros(0, np.complex128))
    with pytest.raises(admm.NumericalError):
        admm.write_cmat(tmp_path / "inf.cmat", np.array([[np.inf + 0j]]))
    with pytest.raises(admm.NumericalError):  # finite in FP64, overflows binary32
        admm.write_cmat(tmp_path / "big.cmat", np.array([[1e300 + 0j]]), dtype="c64")


def test_header_checks(tmp_path):  # cmat_io.hpp:78-100
    def hdr(magic, rows, cols, payload=b""):
        return magic + np.array([rows, cols], "<u8").tobytes() + payload

    for name, data, off in [("zero_rows", hdr(b"CMX1", 0, 3), 4),
                            ("overflow", hdr(b"CMX1", 2**40, 2**40), 4),
                            ("implausible", hdr(b"CMX1", 2**16 + 1, 2**16), 4),
                            ("at_cap_short", hdr(b"CMX1", 2**16, 2**16), 20),
                            ("c64_short", hdr(b"CMF1", 2, 2, bytes(8)), 28)]:
        f = tmp_path / f"{name}.cmat"
        f.write_bytes(data)
        with pytest.raises(admm.FormatError) as e:
            admm.read_cmat(f)
        assert e.value.byte_offset() == off, name
        if not name.startswith("c64"):
            agree(f)
    # a non-finite payload entry: offset of that entry (our reader validates as it streams)
    a = rand_c(3, 3, 38)
    f = tmp_path / "nan.cmat"
    admm.write_cmat(f, a)
    raw = bytearray(f.read_bytes())
    raw[20 + 5 * 16 + 8:20 + 5 * 16 + 16] = np.array([np.nan]).tobytes()
    f.write_bytes(bytes(raw))
    assert agree(f)[0] == ["error", "FormatError", str(20 + 5 * 16)]
