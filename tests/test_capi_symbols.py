"""The C-ABI library loads and exports every symbol include/taskgemm_b200.h declares; host-side
validation mirrors the reference's messages. No compute calls here (CPU)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2203_09353_b200 as tg

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "taskgemm_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:const\s+)?\w+\s*\*?\s*(tg_[a-z0-9_]+)\s*\(", text, re.M)))


def test_header_symbols_exported():
    L = tg.lib()
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert sorted(tg.EXPORTS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", tg.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", tg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", tg.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor op in the shipped kernels


def test_version():
    assert b"sm_100a" in tg.lib().tg_version()


@pytest.mark.parametrize("kw,exc,msg", [
    (dict(spins=1), tg.ConfigError, "spins out of range [2,30]"),
    (dict(spins=40), tg.ConfigError, "spins out of range [2,30]"),
    (dict(procedures=0), tg.ConfigError, "procedures must be >= 1"),
    (dict(devices=0), tg.ConfigError, "devices must be >= 1"),
    (dict(t0=1e-3, t_min=1.0), tg.ConfigError, "anneal schedule requires 0 < t_min <= t0"),
    (dict(t_min=0.0), tg.ConfigError, "anneal schedule requires 0 < t_min <= t0"),
    (dict(spins=26), ValueError, "device tiers cover spins <= 24"),
    (dict(entropy_kind="von-neumann", spins=22), ValueError, "device von-neumann entropy covers spins <= 21"),
    (dict(entropy_kind="tsallis"), tg.ConfigError, "unknown entropy_kind"),
    (dict(shard_index=2, shard_count=2), tg.ConfigError, "shard_index"),
])
def test_validate_messages(kw, exc, msg):
    cfg = tg.ExperimentConfig(**kw)
    with pytest.raises(exc, match=re.escape(msg)):
        cfg.validate()


def test_rows_and_flops():
    assert tg.ExperimentConfig(procedures=10).rows() == 10
    assert tg.ExperimentConfig(procedures=10, shard_index=1, shard_count=4).rows() == 3  # 1,5,9
    assert tg.ExperimentConfig(procedures=10, shard_index=3, shard_count=4).rows() == 2  # 3,7
    assert tg.ExperimentConfig(procedures=2, shard_index=3, shard_count=4).rows() == 0
    # gemm_flops KAT (test_linalg.cpp:281-285): S=21 -> (1024,1024,2048)
    assert tg.step_flops(21) == 17179869184
    assert tg.step_flops(12) == 8 * 64 ** 3
    assert tg.dims_for_spins(15) == (128, 256)


def test_no_cpu_fallback_without_gpu():
    """On a machine without a CUDA device the product path fails loudly."""
    cnt = ctypes.c_int(0)
    try:
        rt = ctypes.CDLL("libcudart.so")
        rc = rt.cudaGetDeviceCount(ctypes.byref(cnt))
    except OSError:
        rc = 1
    if rc == 0 and cnt.value > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(tg.DeviceUnavailable, match="no CUDA device"):
        tg.Device([0])
    with pytest.raises(tg.DeviceUnavailable):
        tg.probe_rng(0, 0, 4)


def test_batched_gemm_contract_errors_host_side():
    import numpy as np
    # fixed-size contract (exec.cpp:156-161) and dims (linalg.cpp:59-73) are checked before any device work
    class Fake(tg.Device):
        def __init__(self):
            self._h = None
    d = Fake()
    with pytest.raises(ValueError, match="non-empty"):
        d.batched_gemm([], [])
    with pytest.raises(ValueError, match="fixed-size"):
        d.batched_gemm([np.zeros((2, 3)), np.zeros((3, 3))], [np.zeros((3, 2)), np.zeros((3, 2))])
    with pytest.raises(ValueError, match=re.escape("A.cols (3) != B.rows (4)")):
        d.batched_gemm([np.zeros((2, 3))], [np.zeros((4, 2))])


@pytest.mark.parametrize("seed,p,init_spins,chunks,extra", [
    (0, 0, -1, 1, 0), (0, 3, -1, 5, 7), (11, 1, -1, 37, 100), (5, 2, 4, 0, 0), (5, 2, 6, 3, 2), (9, 0, 8, 2, 33)])
def test_rng_jump_tables_vs_sequential_stream(oracle, seed, p, init_spins, chunks, extra):
    """The pre-pass's GF(2) jump tables (host copy of what rng_chunk_kernel uploads) land on
    the same xoshiro256++ words as stepping the reference's stream (rng.cpp:23-45) one draw
    at a time: chunk jumps of 34 * tg_rng_chunk_steps() draws and the random-start jump of
    2^(S+1) draws."""
    skip = (2 << init_spins if init_spins >= 0 else 0) + chunks * 34 * int(tg.lib().tg_rng_chunk_steps()) + extra
    want = oracle.first_u64(seed, p, skip + 8)[skip:]
    got = tg.rng_jump_words(seed, p, chunks, extra, 8, init_spins)
    assert np.array_equal(got, want)


def test_environment_switches_documented():
    """Every TG_* environment variable the library reads is listed in DESIGN.md's switch
    table, so no behaviour hides behind an undocumented knob."""
    import glob
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    used = set()
    for path in glob.glob(os.path.join(root, "paper_2203_09353_b200", "csrc", "*")):
        if path.endswith((".cu", ".cuh", ".cpp", ".h")):
            used |= set(re.findall(r'getenv\("(TG_[A-Z0-9_]+)"\)', open(path).read()))
    design = open(os.path.join(root, "DESIGN.md")).read()
    assert used, "no switches found"
    assert not [v for v in sorted(used) if f"`{v}" not in design], sorted(used)


def test_rho_half_validation():
    """rho_half is a Renyi-2 option (both tiers); with von Neumann it is a ConfigError
    (host-side validation, no GPU needed)."""
    for spins in (4, 12, 14, 20):
        tg.ExperimentConfig(spins=spins, steps=2, procedures=1, rho_half=True).validate()
    for bad in (tg.ExperimentConfig(spins=14, steps=2, procedures=1, rho_half=True, entropy_kind="von-neumann"),
                tg.ExperimentConfig(spins=10, steps=2, procedures=1, rho_half=True, entropy_kind="von-neumann")):
        with pytest.raises(tg.ConfigError, match="rho_half"):
            bad.validate()
