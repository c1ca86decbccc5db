"""The device exp (csrc/glibc_exp.cuh) compiled as host C++ must equal the
host libm's exp bit for bit: numpy's ziggurat wedge test compares against
that libm (distributions.c random_standard_exponential).

glibc 2.39 picks its FMA build of exp when the CPU has FMA+AVX2 (the same
condition as log1p); the test uses the variant the engine picks on this host
(cs_host_log1p_variant) and checks 3e7 arguments: the ziggurat's domain
-x, x = ri * we[i] in [0, 7.7), plus random magnitudes in [2^-60, 500].
"""

import hashlib
import os
import subprocess

import pytest

from conftest import ROOT

LIBM = "/lib/x86_64-linux-gnu/libm.so.6"
# this image's libm (glibc 2.39, Ubuntu): entry points of the two exp builds
# the IFUNC resolver __exp_finite chooses between (objdump of the resolver)
LIBM_SHA256 = "3c24a53ee35c2ce0c67240e62bff699c4bddcd7cf8993d5d7ad29157ba072c99"
EXP_SSE2, EXP_FMA = 0x27EA0, 0x79B60

VARIANTS_SRC = r'''
#include <dlfcn.h>
#include <link.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include "glibc_exp.cuh"
static unsigned long long st = 0x2545F4914F6CDD1DULL;
static unsigned long long xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
int main(int argc, char** argv) {
    void* h = dlopen("libm.so.6", RTLD_NOW);
    struct link_map* lm;
    dlinfo(h, RTLD_DI_LINKMAP, &lm);
    double (*v0)(double) = (double (*)(double))((char*)lm->l_addr + strtol(argv[1], 0, 0));
    double (*v1)(double) = (double (*)(double))((char*)lm->l_addr + strtol(argv[2], 0, 0));
    long n = atol(argv[3]), bad = 0;
    for (long i = 0; i < n; i++) {
        unsigned long long w = xr();
        double u = (double)(w >> 11) * (1.0 / 9007199254740992.0);
        double x = -7.7 * u;
        if (i % 5 == 2) x = (xr() & 1 ? 1.0 : -1.0) * 500.0 * u;
        double a0 = v0(x), b0 = cs::glibc_exp(x, 0), a1 = v1(x), b1 = cs::glibc_exp(x, 1);
        bad += memcmp(&a0, &b0, 8) != 0;
        bad += memcmp(&a1, &b1, 8) != 0;
    }
    printf("%ld\n", bad);
    return 0;
}
'''


SRC = r'''
#include "glibc_exp.cuh"
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static unsigned long long st = 0x9E3779B97F4A7C15ULL;
static unsigned long long xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
int main(int argc, char** argv) {
    int variant = atoi(argv[1]);
    long n = atol(argv[2]), bad = 0;
    for (long i = 0; i < n; i++) {
        unsigned long long w = xr();
        double u = (double)(w >> 11) * (1.0 / 9007199254740992.0);
        double x = -7.7 * u;                                        /* the wedge domain */
        if (i % 5 == 1) x = -ldexp(1.0 + u, -(int)(xr() % 60));     /* small magnitudes */
        if (i % 5 == 2) x = (xr() & 1 ? 1.0 : -1.0) * 500.0 * u;    /* the whole main path */
        double a = exp(x), b = cs::glibc_exp(x, variant);
        if (memcmp(&a, &b, 8)) bad++;
    }
    printf("%ld\n", bad);
    return 0;
}
'''


def test_exp_port_matches_libm(tmp_path):
    from paper_2604_14993_b200 import _native as N

    variant = N.load(require_device=False).cs_host_log1p_variant()
    src = tmp_path / "twin.cpp"
    src.write_text(SRC)
    exe = tmp_path / "twin"
    inc = os.path.join(ROOT, "paper_2604_14993_b200", "csrc")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", inc, str(src), "-o", str(exe), "-lm"],
                   check=True)
    for v in sorted({variant, 1 - variant}):
        out = subprocess.run([str(exe), str(v), "30000000"], capture_output=True, text=True, check=True)
        bad = int(out.stdout.strip())
        if v == variant:  # the variant this host's libm runs
            assert bad == 0, (v, bad)
        else:  # the other build differs from this libm in the last bit now and then
            assert bad < 30000000 // 100, (v, bad)


def test_exp_port_matches_both_libm_builds(tmp_path):
    """Both builds (FMA and SSE2) against the libm's own entry points, when
    this is the image's libm (their addresses are build specific)."""
    if hashlib.sha256(open(LIBM, "rb").read()).hexdigest() != LIBM_SHA256:
        pytest.skip("not this image's libm build")
    src = tmp_path / "variants.cpp"
    src.write_text(VARIANTS_SRC)
    exe = tmp_path / "variants"
    inc = os.path.join(ROOT, "paper_2604_14993_b200", "csrc")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", inc, str(src), "-o", str(exe), "-ldl", "-lm"],
                   check=True)
    out = subprocess.run([str(exe), hex(EXP_SSE2), hex(EXP_FMA), "20000000"], capture_output=True, text=True,
                         check=True)
    assert int(out.stdout.strip()) == 0
