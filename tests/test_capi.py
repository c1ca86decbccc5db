"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/chainserve_b200.h declares, the host-side key derivation is
numpy-exact, and compute entry points refuse to run without a device (no CPU
fallback)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "chainserve_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_14993_b200 import _native as N

    return N.load(require_device=False)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("cs_philox_keys", "cs_exp_streams", "cs_jffc_sim", "cs_rep_stats", "cs_run_sim_host",
              "cs_gbp_batch", "cs_gca_batch"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2604_14993_b200 import _native as N

    assert set(N.EXPORTS) <= set(declared_symbols())


def test_version_and_log1p_variant(lib):
    assert lib.cs_version().startswith(b"chainserve_b200")
    assert lib.cs_host_log1p_variant() in (0, 1)


def test_host_philox_keys_match_golden(lib, golden):
    from paper_2604_14993_b200 import _native as N

    meta, arr = golden
    for (seed, rep), key in zip(meta["rng_key_cases"], arr["rng_keys"]):
        w = N.seed_words(seed)
        reps = np.array([rep], np.uint64)
        out = np.zeros(2, np.uint64)
        st = lib.cs_philox_keys(N.ptr(w, C.c_uint32), len(w), N.ptr(reps, C.c_uint64), 1,
                                N.ptr(out, C.c_uint64))
        assert st == 0 and np.array_equal(out, key), (seed, rep)


def test_compute_calls_refuse_without_device(lib):
    from paper_2604_14993_b200 import _native as N

    if lib.cs_device_count() > 0:
        pytest.skip("a CUDA device is present")
    assert lib.cs_exp_streams(None, 1, 1, None, 1, 1, None) == N.CS_ERR_CUDA
    import paper_2604_14993_b200 as P

    with pytest.raises(N.NativeUnavailable):
        P.run_sim(P.SimConfig(rates=(1.0,), capacities=(1,), workload=P.PoissonWorkload(0.5),
                              horizon_jobs=10))


def test_struct_layouts_match_header():
    from paper_2604_14993_b200 import _native as N

    assert C.sizeof(N.SimPoint) == 16
    assert C.sizeof(N.RepSummary) == 16 * 8
    assert C.sizeof(N.ComposePoint) == 8 + 4 * 8 + 16
