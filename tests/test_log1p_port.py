"""The device log1p (csrc/glibc_log1p.cuh) compiled as host C++ must equal the
host libm's log1p bit for bit: numpy's ziggurat tail calls that libm.

glibc 2.39 picks its FMA build of log1p when the CPU has FMA+AVX2; the test
uses the same variant the engine would pick on this host
(cs_host_log1p_variant) and checks ~2e7 inputs from the ziggurat domain
x = -u, u = k * 2^-53, plus positive and tiny arguments.
"""

import os
import subprocess

import pytest

from conftest import ROOT

SRC = r'''
#include "glibc_log1p.cuh"
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static unsigned long long st = 88172645463325252ULL;
static unsigned long long xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
int main(int argc, char** argv) {
    int variant = atoi(argv[1]);
    long n = atol(argv[2]), bad = 0;
    for (long i = 0; i < n; i++) {
        unsigned long long w = xr();
        double u = (double)(w >> 11) * (1.0 / 9007199254740992.0);
        if (i % 4 == 1) u = (double)(w >> 40) * (1.0 / 9007199254740992.0);
        if (i % 4 == 2) u = ldexp((double)(w >> 11), -53 - (int)(xr() % 40));
        double x = -u;
        if (i % 8 == 3) x = ldexp((double)(w >> 11), -53 + (int)(xr() % 60));
        double a = log1p(x), b = cs::glibc_log1p(x, variant);
        if (memcmp(&a, &b, 8)) bad++;
    }
    printf("%ld\n", bad);
    return 0;
}
'''


def test_log1p_port_matches_libm(tmp_path):
    from paper_2604_14993_b200 import _native as N

    variant = N.load(require_device=False).cs_host_log1p_variant()
    src = tmp_path / "twin.cpp"
    src.write_text(SRC)
    exe = tmp_path / "twin"
    inc = os.path.join(ROOT, "paper_2604_14993_b200", "csrc")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", inc, str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), str(variant), "20000000"], capture_output=True, text=True,
                         check=True)
    assert int(out.stdout.strip()) == 0
