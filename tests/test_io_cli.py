"""TLT1 container, P6 frame directories and the CLI, mirroring the
reference's tests/test_io_cli.py: host-side parts run on the CPU, numeric commands and the
device payload reorder on the GPU.  The container byte stream is pinned to files the
reference itself wrote (tests/golden: io_*)."""

import numpy as np
import pytest

from paper_2202_02870_b200 import io as tio
from paper_2202_02870_b200.cli import main
from paper_2202_02870_b200.completion import sample_mask
from paper_2202_02870_b200.errors import FormatError


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.mark.parametrize("name", ["io_f64", "io_f32", "io_c128", "io_mask"])
def test_container_bytes_match_reference(golden, tmp_path, name):
    x = golden[f"{name}/x"]
    path = tmp_path / "x.tlt"
    tio.write_container(path, x)
    assert path.read_bytes() == golden[f"{name}/bytes"].tobytes()
    back = tio.read_container(path)
    assert back.dtype == x.dtype and back.flags.c_contiguous
    np.testing.assert_array_equal(back, x)


def test_roundtrips_and_determinism(tmp_path, rng):
    for x in (rng.standard_normal((3, 4, 2, 5)), rng.standard_normal((2, 3, 4)).astype(np.float32),
              rng.standard_normal((2, 2, 3)) + 1j * rng.standard_normal((2, 2, 3)), sample_mask((5, 4, 3, 2), 0.37, 21)):
        a, b = tmp_path / "a.tlt", tmp_path / "b.tlt"
        tio.write_container(a, x)
        tio.write_container(b, x)
        assert a.read_bytes() == b.read_bytes()
        np.testing.assert_array_equal(tio.read_container(a), x)


def test_container_errors(tmp_path, rng):
    bad = tmp_path / "bad.tlt"
    bad.write_bytes(b"NOPE" + bytes(16))
    with pytest.raises(FormatError, match="magic"):
        tio.read_container(bad)
    x = rng.standard_normal((2, 2, 2))
    p = tmp_path / "x.tlt"
    tio.write_container(p, x)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(FormatError, match="payload length 56 bytes"):
        tio.read_container(p)
    p.write_bytes(b"TLT1" + bytes([9]) + bytes(80))
    with pytest.raises(FormatError, match="unsupported order 9"):
        tio.read_container(p)
    with pytest.raises(FormatError, match="orders 2..8"):
        tio.write_container(p, np.zeros(3))
    p.write_bytes(b"TLT1" + bytes([2]) + np.array([1, 1], "<u8").tobytes() + bytes([7]) + bytes(8))
    with pytest.raises(FormatError, match="dtype code 7"):
        tio.read_container(p)


def test_ppm_roundtrip_and_guards(tmp_path, rng):
    x = np.round(rng.random((4, 5, 3, 3)) * 255) / 255
    tio.export_ppm_dir(x, tmp_path / "v")
    np.testing.assert_array_equal(tio.import_ppm_dir(tmp_path / "v"), x)
    assert sorted(p.name for p in (tmp_path / "v").iterdir())[0] == "frame_0000.ppm"
    (tmp_path / "c").mkdir()
    (tmp_path / "c" / "a.ppm").write_bytes(b"P6\n# comment\n1 1\n255\n" + bytes([255, 255, 255]))
    np.testing.assert_array_equal(tio.import_ppm_dir(tmp_path / "c"), np.ones((1, 1, 3, 1)))
    (tmp_path / "c" / "b.ppm").write_bytes(b"P5\n1 1\n255\n" + bytes([1]))
    with pytest.raises(FormatError, match="P6"):
        tio.import_ppm_dir(tmp_path / "c")
    (tmp_path / "e").mkdir()
    with pytest.raises(FormatError, match="no .ppm"):
        tio.import_ppm_dir(tmp_path / "e")
    with pytest.raises(FormatError, match="H x W x 3 x T"):
        tio.export_ppm_dir(np.zeros((2, 2, 2, 2)), tmp_path / "z")


def test_cli_host_commands(tmp_path, capsys):
    a, b = tmp_path / "a.tlt", tmp_path / "b.tlt"
    for out in (a, b):
        assert main(["mask", "gen", "--dims", "6,6,3", "--sr", "0.4", "--seed", "5", "--out", str(out)]) == 0
    assert a.read_bytes() == b.read_bytes()
    mask = tio.read_container(a)
    assert mask.dtype == bool and mask.sum() == round(0.4 * 108)
    assert main(["mask", "gen", "--bogus", "1"]) == 1
    assert main([]) == 1
    assert main(["metrics", "--a", str(tmp_path / "nope.tlt"), "--b", str(tmp_path / "nope.tlt")]) == 2


# ---------------------------------------------------------------- GPU: numeric commands
@pytest.mark.gpu
def test_cli_numeric_commands(tmp_path, capsys, rng):
    import paper_2202_02870_b200 as L

    a = rng.standard_normal((2, 3, 2, 2))
    b = rng.standard_normal((3, 2, 2, 2))
    pa, pb, po = tmp_path / "a.tlt", tmp_path / "b.tlt", tmp_path / "o.tlt"
    tio.write_container(pa, a)
    tio.write_container(pb, b)
    assert main(["product", "--a", str(pa), "--b", str(pb), "--transform", "dct", "--out", str(po)]) == 0
    np.testing.assert_allclose(tio.read_container(po), L.l_product(a, b, L.make_spec("dct", (2, 2, 2, 2))),
                               atol=1e-12)
    x = rng.standard_normal((3, 3, 2, 2))
    tio.write_container(pa, x)
    pu, ps, pv = (tmp_path / n for n in ("u.tlt", "s.tlt", "v.tlt"))
    assert main(["tsvd", "--input", str(pa), "--transform", "fft", "--out-u", str(pu), "--out-s", str(ps),
                 "--out-v", str(pv)]) == 0
    u, s, v = (tio.read_container(p) for p in (pu, ps, pv))
    spec = L.make_spec("fft", x.shape)
    np.testing.assert_allclose(L.l_product(L.l_product(u, s, spec), L.l_transpose(v, spec), spec), x, atol=1e-9)
    assert main(["svt", "--input", str(pa), "--tau", "0.5", "--transform", "dct", "--out", str(po)]) == 0
    np.testing.assert_allclose(tio.read_container(po), L.svt(x, 0.5, L.make_spec("dct", x.shape)), atol=1e-12)
    assert main(["metrics", "--a", str(pa), "--b", str(pa)]) == 0
    out = capsys.readouterr().out
    assert "RSE 0" in out and "PSNR inf" in out


@pytest.mark.gpu
def test_cli_complete(tmp_path, capsys, rng):
    import paper_2202_02870_b200 as L

    dims = (16, 16, 3)
    spec = L.make_spec("fft", dims)
    m = L.l_product(rng.standard_normal((16, 2, 3)), rng.standard_normal((2, 16, 3)), spec)
    pm, pk, po, pt = (tmp_path / n for n in ("m.tlt", "mask.tlt", "out.tlt", "trace.csv"))
    tio.write_container(pm, m)
    tio.write_container(pk, sample_mask(dims, 0.6, 2))
    code = main(["complete", "--input", str(pm), "--mask", str(pk), "--transform", "fft", "--max-iters", "300",
                 "--tol", "1e-6", "--mu-bar-ratio", "1e-6", "--ground-truth", str(pm), "--trace-csv", str(pt),
                 "--out", str(po)])
    out = capsys.readouterr().out
    assert code == 0 and "status" in out and "RSE" in out
    assert pt.read_text().startswith("iter,mu,t,rel_change,rse,psnr")
    assert L.rse(tio.read_container(po), m) < 1e-2
    x = rng.standard_normal((4, 4, 2))
    tio.write_container(pm, x)
    tio.write_container(pk, sample_mask((4, 4, 2), 0.5, 1))
    assert main(["complete", "--input", str(pm), "--mask", str(pk), "--transform", "cprod", "--out",
                 str(tmp_path / "o2.tlt")]) == 2
    assert "unitary-scaled" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["io_f64", "io_f32", "io_c128"])
def test_read_container_device(golden, tmp_path, name):
    """The column-major payload reordered to C order on the GPU equals the host read, bit for bit."""
    p = tmp_path / "x.tlt"
    p.write_bytes(golden[f"{name}/bytes"].tobytes())
    d = tio.read_container_device(p)
    np.testing.assert_array_equal(d.numpy(), golden[f"{name}/x"])
    with pytest.raises(FormatError):
        q = tmp_path / "m.tlt"
        q.write_bytes(golden["io_mask/bytes"].tobytes())
        tio.read_container_device(q)
