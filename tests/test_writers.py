"""§8(f)-4 writers: the native surface-CSV formatter is byte-identical to the
reference's _write_csv (cli.py:83-90) with repr() floats, on edge values and a
realistic dB map; the full ambiguity output set matches the reference's files
(except the manifest timestamp).  CPU only (host code in libsignadd_b200.so)."""

import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


@pytest.fixture(scope="module")
def cli():
    for c in REF_CANDIDATES:
        if os.path.isdir(os.path.join(c, "signadd")):
            if c not in sys.path:
                sys.path.insert(0, c)
            import signadd.cli as m
            return m
    pytest.skip("reference package not available")


EDGE = [0.0, -0.0, 1.0, -1.0, 0.1, -300.0, 1e16, 9999999999999998.0, 1e15, 123456789012345678.0, 1e-4, 1e-5,
        0.00012345, -1.5e-7, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, math.pi, -math.e * 1e-3,
        100.0, 1e22, 1e-300, -12.345678901234567, 0.5, 2.0 ** 60, 3.0e10, float("inf"), float("-inf")]


def test_float_repr_edges():
    from paper_1402_0532_b200.writers import format_float_repr
    for v in EDGE:
        assert format_float_repr(v) == repr(float(v)), v
    assert format_float_repr(float("nan")) == "nan"
    g = np.random.default_rng(3)
    for v in np.concatenate([g.standard_normal(2000) * 10.0 ** g.integers(-20, 20, 2000), -300 * g.random(2000)]):
        assert format_float_repr(v) == repr(float(v))


def test_surface_csv_byte_identical(cli, tmp_path):
    from paper_1402_0532_b200.writers import magnitude_db, surface_csv_bytes
    g = np.random.default_rng(11)
    vals = (g.standard_normal((37, 64)) + 1j * g.standard_normal((37, 64))) * np.exp(-g.random((37, 64)) * 20)
    vals[3, 5] = 0  # -> floor -300.0
    db = magnitude_db(vals)
    want_path = str(tmp_path / "ref.surface.csv")
    cli._write_csv(want_path, ["l", "p", "magnitude_db"],
                   ((l, p, float(db[l, p])) for l in range(db.shape[0]) for p in range(db.shape[1])),
                   "x.manifest.json")
    want = open(want_path, "rb").read()
    for nt in (1, 3, 8):
        assert surface_csv_bytes(db, "x.manifest.json", nt) == want
    # a map large enough for the threaded path, against a direct restatement
    big = -300.0 * g.random((300, 512))
    big[0, 0] = 0.0
    got = surface_csv_bytes(big, "m.json", 4)
    lines = got.decode().split("\n")
    assert lines[0] == "# manifest=m.json" and lines[1] == "l,p,magnitude_db"
    for c in (0, 1, 511, 512, 150000, 300 * 512 - 1):
        assert lines[2 + c] == f"{c // 512},{c % 512},{repr(float(big.flat[c]))}"


def test_ambiguity_outputs_match_reference_cli(cli, tmp_path):
    """The output set of `signadd ambiguity` for one surface: surface, range and
    Doppler cuts byte-identical to the reference's writers."""
    import signadd
    from paper_1402_0532_b200.writers import write_ambiguity_outputs
    g = np.random.default_rng(5)
    vals = g.standard_normal((16, 32)) + 1j * g.standard_normal((16, 32))
    sf = signadd.AmbiguitySurface(values=vals, range_bin_m=1500.0, doppler_bin_hz=6.25,
                                  variant=signadd.AmbiguityVariant.EQ12A, sample_rate_hz=200000.0)
    args = {"variant": "eq12a", "seed": 7}
    paths = write_ambiguity_outputs(str(tmp_path / "ours"), sf, args)
    ref = str(tmp_path / "ref")
    man = cli._write_manifest(ref, "ambiguity", args, sf.op_counts)
    db = sf.magnitude_db()
    cli._write_csv(ref + ".surface.csv", ["l", "p", "magnitude_db"],
                   ((l, p, float(db[l, p])) for l in range(sf.l_bins) for p in range(sf.n)), man)
    ls, rk, rdb = sf.range_cut()
    cli._write_csv(ref + ".range_cut.csv", ["l", "bistatic_range_km", "magnitude_db"],
                   [(int(l), float(r), float(v)) for l, r, v in zip(ls, rk, rdb)], man)
    fr, cdb = sf.doppler_cut()
    cli._write_csv(ref + ".doppler_cut.csv", ["doppler_hz", "magnitude_db"],
                   [(float(f), float(v)) for f, v in zip(fr, cdb)], man)
    for kind in ("surface", "range_cut", "doppler_cut"):
        a = open(paths[kind], "rb").read().replace(b"ours.manifest.json", b"M")
        b = open(ref + f".{kind}.csv", "rb").read().replace(b"ref.manifest.json", b"M")
        assert a == b, kind
