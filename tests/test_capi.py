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


def test_extended_entry_points_are_declared():
    syms = declared_symbols()
    for s in ("cs_occupancy_bounds", "cs_birth_death_occupancy", "cs_sim_ext", "cs_ragged_rows"):
        assert s in syms


def test_extended_calls_refuse_without_device(lib):
    from paper_2604_14993_b200 import _native as N

    if lib.cs_device_count() > 0:
        pytest.skip("a CUDA device is present")
    assert lib.cs_occupancy_bounds(None, 1, None, None, 1, None, None, None) == N.CS_ERR_CUDA
    assert lib.cs_birth_death_occupancy(None, 1, None, 1, None, None, None) == N.CS_ERR_CUDA
    assert lib.cs_sim_ext(None, None) == N.CS_ERR_CUDA
    assert lib.cs_ragged_rows(None, 1, 1, None, None, None) == N.CS_ERR_CUDA


def test_ctypes_layouts_match_the_c_compiler(tmp_path):
    """sizeof/offsetof of the boundary structs as gcc lays them out from
    include/chainserve_b200.h == the ctypes mirrors in _native / sim_ext."""
    import shutil
    import subprocess

    from paper_2604_14993_b200 import _native as N
    from paper_2604_14993_b200.sim_ext import ExtArgs

    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    fields = [f for f, _ in ExtArgs._fields_]
    src = tmp_path / "layout.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "chainserve_b200.h"', "int main(void) {",
             'printf("%zu %zu %zu %zu %zu\\n", sizeof(cs_sim_ext_args), sizeof(cs_bounds_out), '
             'sizeof(cs_bound_point), sizeof(cs_bd_point), sizeof(cs_rep_summary));']
    for f in fields:
        lines.append(f'printf("%zu\\n", offsetof(cs_sim_ext_args, {f}));')
    lines.append("return 0; }")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out[:5]]
    assert sizes == [C.sizeof(ExtArgs), N.BOUNDS_DTYPE.itemsize, C.sizeof(N.BoundPoint),
                     C.sizeof(N.BdPoint), C.sizeof(N.RepSummary)]
    assert [int(x) for x in out[5:]] == [getattr(ExtArgs, f).offset for f in fields]
