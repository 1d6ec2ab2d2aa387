"""CPU-only checks: the C-ABI library loads and exports every symbol the header
declares; host-side logic (twiddles, contracts, counts, workloads) matches the
reference.  No kernel is launched here."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "signadd_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|void|const char \*)\s*(sa_\w+)\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_1402_0532_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_native.SIGNATURES) == syms
    assert _native.lib().sa_version() == 1


def test_library_is_sm100a():
    import subprocess
    from paper_1402_0532_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_twiddles_match_reference_pin(golden):
    import paper_1402_0532_b200 as sa
    for n, h in zip(golden["tw_sizes"], golden["tw_sha"]):
        assert hashlib.sha256(sa.twiddle_table(int(n)).entries.tobytes()).hexdigest() == str(h)
    assert sa.unit_tone(7, 64)[32] == complex(-1.0, 0.0)


def test_contracts_raise_before_device():
    import paper_1402_0532_b200 as sa
    for n in (1, 3, 12, 100):
        with pytest.raises(sa.ContractError):
            sa.nfft(np.ones(n, complex))
    with pytest.raises(sa.ContractError):
        sa.ndft(np.ones((2, 2), complex))
    with pytest.raises(sa.ContractError):
        sa.ndft([])
    with pytest.raises(sa.DomainError):
        sa.ndft([np.nan, 1])
    with pytest.raises(sa.ContractError):
        sa.lag_product_mf(np.ones(8, complex), np.ones(8, complex), 8)
    with pytest.raises(sa.ContractError):
        sa.lag_product_mf(np.ones(8, complex), np.ones(8, complex), -1)
    with pytest.raises(sa.ContractError):
        sa.lag_product_mf(np.ones(4, complex), np.ones(8, complex), 0, n=8)
    with pytest.raises(ValueError):  # the reference crashes with a numpy ValueError for l > n
        sa.lag_product_mf(np.ones(8, complex), np.ones(16, complex), 10, n=8)
    with pytest.raises(sa.ContractError):
        sa.ComplexSignal(np.ones(4), 0.0)
    S = sa.ComplexSignal
    with pytest.raises(sa.ContractError):
        sa.ambiguity_eq12a(np.ones(8), np.ones(8), 2, 8)  # no sample rate
    with pytest.raises(sa.ContractError):
        sa.ambiguity_eq12a(S(np.ones(8), 1.0), S(np.ones(8), 2.0), 2, 8)
    with pytest.raises(sa.ContractError):
        sa.ambiguity_eq12a(S(np.ones(8), 1.0), S(np.ones(8), 1.0), 0, 8)
    for var in ("eq11", "eq12b", "eq12c"):  # exact-multiply variants: same contracts
        with pytest.raises(sa.ContractError, match="power of two"):
            sa.compute_ambiguity(var, S(np.ones(12), 1.0), S(np.ones(12), 1.0), 2, 12)
        with pytest.raises(sa.ContractError):
            sa.compute_ambiguity(var, S(np.ones(8), 1.0), S(np.ones(8), 1.0), 9, 8)
    for n in (1, 3, 12):
        with pytest.raises(sa.ContractError, match="fft_exact"):
            sa.fft_exact(np.ones(n, complex))
    with pytest.raises(sa.ContractError):
        sa.lag_product_exact(np.ones(8, complex), np.ones(8, complex), 8)


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_1402_0532_b200 as sa
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        sa.ndft(np.ones(4, complex))
    with pytest.raises(RuntimeError, match="CUDA"):
        sa.nfft_batch(np.ones((2, 4), complex))


def test_count_formulas():
    import paper_1402_0532_b200 as sa
    for n in (2, 4, 8, 1024, 65536):
        lg = int(np.log2(n))
        assert sa.nfft_complex_ops(n) == n * (lg + 1) == 4 * (n // 2) + 2 * (sa.nfft_butterflies(n) - n // 2)
        assert sa.ndft_complex_ops(n) == n * n
    assert sa.nfft_dif_complex_ops(65536) == 622592
    assert sa.map_complex_ops(1024, 1 << 20, 512) == 1024 * (1 << 20) + 1024 * 512 * 10
    c = sa.OpCounter()
    c.count_complex(7)
    r = c.report()
    assert (r.sign_ops, r.abs_ops, r.add_ops, r.complex_mf_ops) == (28, 56, 42, 7)


def test_workload_generators():
    from paper_1402_0532_b200 import workloads as w
    x = w.c1_ndft64(16)
    assert x.shape == (17, 64) and np.array_equal(x[0], w.unit_tone(7, 64))
    a = w.c3_nlfft_rows(256, np.array([3, 5]))
    b = w.c3_nlfft_rows(256, np.array([5]))
    assert np.array_equal(a[1], b[0])
    sc = w.radar_scene(1 << 12, 3, 1)
    assert sc.surv.shape == sc.ref.shape == (1 << 12,)
    assert np.allclose(np.abs(sc.ref), 1.0)
    assert np.all((sc.delays >= 10) & (sc.delays <= 900))


def test_oracle_not_imported_by_product():
    import subprocess
    import sys
    code = ("import sys; import paper_1402_0532_b200, paper_1402_0532_b200.sharded, "
            "paper_1402_0532_b200.workloads; print('oracle' in sys.modules)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.strip() == "False", out.stderr
    for dp, _, files in os.walk(os.path.join(ROOT, "paper_1402_0532_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f
