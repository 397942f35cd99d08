"""CCF1 FieldFile I/O through the C-ABI, host paths (no GPU): format, CRC-32 and the reference's
error behaviour (proj/src/io.cpp:12-109, proj/include/cylspec/io.hpp:11-28). The reference's own
test_io.cpp is a placeholder; the CRC is pinned to the published CRC-32/IEEE check value, to
zlib.crc32 and to the oracle's restatement of crc32_ieee (io.cpp:12-25)."""
import struct
import zlib

import numpy as np
import pytest


def test_crc32_known_answers(P, O):
    assert P.crc32(b"123456789") == 0xCBF43926  # CRC-32/IEEE check value
    assert P.crc32(b"") == 0
    rng = np.random.default_rng(0)
    for n in [1, 3, 7, 8, 9, 63, 64, 65, 1000, 16384, 16391, 100003]:
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert P.crc32(b) == zlib.crc32(b) == O.crc32(b), n


def _parse(raw):
    assert raw[:4] == b"CCF1"
    version, = struct.unpack("<I", raw[4:8])
    kind = raw[8]
    m, n, p = struct.unpack("<III", raw[9:21])
    payload = raw[21:-4]
    crc, = struct.unpack("<I", raw[-4:])
    return version, kind, (m, n, p), payload, crc


@pytest.mark.parametrize("kind", [0, 1])
def test_write_read_round_trip(P, tmp_path, kind):
    rng = np.random.default_rng(kind)
    p, n, m = 8, 6, 4
    a = rng.standard_normal((p, n, m))
    if kind:
        a = a + 1j * rng.standard_normal((p, n, m))
    path = tmp_path / "f.ccf"
    P.write_field(path, a)
    version, k, shape, payload, crc = _parse(path.read_bytes())
    assert (version, k, shape) == (1, kind, (m, n, p))
    assert crc == zlib.crc32(payload)
    assert np.array_equal(np.frombuffer(payload, "<f8").view(a.dtype).reshape(a.shape), a)
    assert P.read_field_header(path) == dict(kind=kind, m=m, n=n, p=p)
    b = P.read_field(path)
    assert b.dtype == a.dtype and np.array_equal(a, b)


def test_reference_error_messages(P, tmp_path):
    a = np.arange(4 * 4 * 2, dtype=np.float64).reshape(2, 4, 4)
    good = tmp_path / "g.ccf"
    P.write_field(good, a)
    raw = good.read_bytes()

    def bad(data, msg):
        f = tmp_path / "b.ccf"
        f.write_bytes(data)
        with pytest.raises(P.FieldFileError, match=msg):
            P.read_field(f)

    bad(b"XCF1" + raw[4:], "bad magic")
    bad(raw[:4] + struct.pack("<I", 2) + raw[8:], "unsupported version 2")
    bad(raw[:8] + bytes([5]) + raw[9:], "unknown kind")
    bad(raw[:15], "truncated header")
    bad(raw[:40], "truncated payload")
    bad(raw[:-2], "truncated header")  # the CRC word is read like a header field (io.cpp:31-38)
    flip = bytearray(raw)
    flip[30] ^= 0x10
    bad(bytes(flip), "CRC mismatch")
    with pytest.raises(P.FieldFileError, match="cannot open"):
        P.read_field(tmp_path / "missing.ccf")
    with pytest.raises(P.DomainError):  # GridSpec::validate (grid.cpp:8-14)
        bad_spec = raw[:9] + struct.pack("<III", 3, 4, 2) + raw[21:]
        f = tmp_path / "s.ccf"
        f.write_bytes(bad_spec)
        P.read_field(f)
    with pytest.raises(P.FieldFileError, match="cannot open for writing"):
        P.write_field(tmp_path / "no" / "such" / "dir.ccf", a)
