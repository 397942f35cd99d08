"""GPU paths of the CCF1 FieldFile I/O: the device CRC-32 (parallel chunk CRCs merged by GF(2)
shifts, csrc/fieldio.cu) against zlib at awkward sizes, device-resident write / read, and NS
snapshots written straight from the device state (cylspec_main.cpp:111-113)."""
import zlib

import numpy as np
import pytest
import torch

from tests.inputs import hermitian_coeffs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes", [8, 64, 16376, 16384, 16392, 4194304 + 24, 67108864 + 8 * 1001])
def test_device_crc_matches_zlib(P, nbytes):
    rng = np.random.default_rng(nbytes)
    host = rng.integers(0, 256, nbytes, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    assert P.crc32(dev) == zlib.crc32(host.tobytes())


def test_device_write_read(P, tmp_path):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((16, 12, 10)) + 1j * rng.standard_normal((16, 12, 10))
    P.write_field(tmp_path / "h.ccf", a)
    P.write_field(tmp_path / "d.ccf", torch.from_numpy(a).cuda())
    assert (tmp_path / "h.ccf").read_bytes() == (tmp_path / "d.ccf").read_bytes()
    out = torch.zeros(16, 12, 10, dtype=torch.complex128, device="cuda")
    P.read_field(tmp_path / "h.ccf", out)
    assert np.array_equal(out.cpu().numpy(), a)
    raw = bytearray((tmp_path / "h.ccf").read_bytes())
    raw[100] ^= 1
    (tmp_path / "x.ccf").write_bytes(bytes(raw))
    with pytest.raises(P.FieldFileError, match="CRC mismatch"):
        P.read_field(tmp_path / "x.ccf", out)  # checked on the GPU


def test_ns_snapshot_from_device(P, tmp_path):
    m = n = p = 32
    ctx = P.Context(m, n, p)
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 3), hermitian_coeffs(m, n, p, 0.7, 103)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    st.step(6)
    wl, wg = st.omega()
    st.write_omega(tmp_path / "lam.ccf", tmp_path / "gam.ccf")
    assert np.array_equal(P.read_field(tmp_path / "lam.ccf"), wl)
    assert np.array_equal(P.read_field(tmp_path / "gam.ccf"), wg)
    assert P.read_field_header(tmp_path / "lam.ccf") == dict(kind=1, m=m, n=n, p=p)
    # a snapshot is a valid initial condition (the CLI's --init path): restart continues identically
    st2 = P.NSStepper(ctx, P.read_field(tmp_path / "lam.ccf"), P.read_field(tmp_path / "gam.ccf"),
                      reynolds=100.0, h=1e-3)
    assert np.isfinite(st2.omega()[0]).all()
    st2.close()
    st.close()
    ctx.close()
