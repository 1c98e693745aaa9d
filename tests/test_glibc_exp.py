"""The device exp (csrc/glibc_exp.cuh) restates glibc's exp operation for operation; its host
build must be bit-identical to the libm exp() the reference's std::exp calls (sample_token,
include/sgrpo/tinylm.hpp:614-627), over 2^24 random + special arguments."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cpu_has_fma_avx2():
    try:
        flags = open("/proc/cpuinfo").read().split()
    except OSError:
        return False
    return "fma" in flags and "avx2" in flags


@pytest.mark.skipif(not _cpu_has_fma_avx2(), reason="libm picks its non-FMA exp variant on this CPU")
def test_host_restatement_bit_identical_to_libm(tmp_path):
    exe = tmp_path / "gx"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "paper_2509_21792_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "glibc_exp_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    n, bad = map(int, r.stdout.strip().splitlines()[-1].split())
    assert n > 16_000_000
    assert bad == 0, r.stdout


def test_generated_table_matches_this_libm():
    """glibc_exp_data.h is what scripts/gen_glibc_exp.py extracts from this image's libm."""
    import importlib.util
    import tempfile
    spec = importlib.util.spec_from_file_location("gen", os.path.join(ROOT, "scripts", "gen_glibc_exp.py"))
    committed = open(os.path.join(ROOT, "paper_2509_21792_b200", "csrc", "glibc_exp_data.h")).read()
    with tempfile.TemporaryDirectory() as d:
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.OUT = os.path.join(d, "x.h")
        mod.main()
        assert open(mod.OUT).read() == committed
