"""CPU checks of the glibc port behind the on-device sampler.

The device sampler (csrc/bmc_sampler.cu) replays glibc 2.39's FMA libm
variants (__log_fma, __cos_fma, __sin_fma) op for op from csrc/bmc_libm.h.
The same header, compiled for the host with single-rounding ops, must equal
the live host libm bit for bit on every argument the reference sampler can
produce (sampling.cpp:48-53, dynamics.cpp:64) -- this is the gate
bmc_device_sampler_available() applies at run time.  The GPU half
(device == host port == reference draw_batch) is tests/test_gpu_sampler.py.
"""
import hashlib
import os

import numpy as np
import pytest

import paper_2604_27193_b200 as bmc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["log", "log near 1", "cos(2 pi u)", "sin |x|<=1.5", "sin/cos reduced", "normal deviate",
         "boundaries"]


@pytest.mark.parametrize("seed", [3, 0x5eed, 2**63 + 11])
def test_port_equals_host_libm(seed):
    mism = bmc.libm_selftest(1 << 21, seed)
    assert mism.tolist() == [0] * 7, dict(zip(NAMES, mism.tolist()))


def test_port_covers_the_seed3_reference_stream():
    # the first 4M normal deviates of the default seed (= the deviates of the
    # first 800k samples of draw_batch(UncertaintyModel{}, .))
    mism = bmc.libm_selftest(1 << 22, 3)
    assert int(mism[5]) == 0 and mism.sum() == 0


def test_device_sampler_gate_passes_on_this_host():
    assert bmc.device_sampler_available()


def test_tables_extracted_from_this_libm():
    hdr = open(os.path.join(ROOT, "paper_2604_27193_b200", "csrc", "bmc_glibc_tables.h")).read()
    libm = "/lib/x86_64-linux-gnu/libm.so.6"
    if not os.path.exists(libm):
        pytest.skip("no x86-64 glibc libm here")
    sha = hashlib.sha256(open(libm, "rb").read()).hexdigest()
    assert f'"{sha}"' in hdr
