"""The reference's own encoder, compiled unmodified from its sources, runs its
2-layer forward + backward with the B200 operator interposed under its
cosine_attention_fused / cosine_attention_backward symbols (tests/cpp).
CPU part: the wiring (exports, link order, PLT calls).  GPU part: the
interposed run equals the pure-reference run."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
ADAPTER = os.path.join(ROOT, "paper_2602_06935_b200", "host", "libcotten_cosrec.so")
REFLIB = os.path.join(ROOT, "oracle", "_ref", "libcosrec_model.so")
FUSED = "_ZN6cosrec22cosine_attention_fusedERKNS_6MatrixES2_S2_dRKNS_15AttentionConfigEPNS_14AttentionCacheEPKNS_7RowMaskE"
BACKWARD = "_ZN6cosrec25cosine_attention_backwardERKNS_14AttentionCacheERKNS_6MatrixE"

needs_build = pytest.mark.skipif(not os.path.exists(os.path.join(BUILD, "dropin_gpu")),
                                 reason="tests/cpp not built (needs /root/reference headers)")


@needs_build
def test_adapter_exports_the_reference_signatures():
    out = subprocess.run(["nm", "-D", "--defined-only", ADAPTER], capture_output=True, text=True,
                         check=True).stdout
    assert re.search(r"\bT " + FUSED + r"\b", out)
    assert re.search(r"\bT " + BACKWARD + r"\b", out)


@needs_build
def test_reference_calls_the_operator_through_the_plt():
    dis = subprocess.run(["objdump", "-d", "--no-show-raw-insn", REFLIB], capture_output=True,
                         text=True, check=True).stdout
    assert re.search(r"call.*<" + FUSED + "@plt>", dis)
    assert re.search(r"call.*<" + BACKWARD + "@plt>", dis)


@needs_build
def test_adapter_is_loaded_ahead_of_the_reference():
    out = subprocess.run(["readelf", "-d", os.path.join(BUILD, "dropin_gpu")], capture_output=True,
                         text=True, check=True).stdout
    needed = re.findall(r"\[(lib[^\]]+)\]", out)
    assert needed.index("libcotten_cosrec.so") < needed.index("libcosrec_model.so")


@needs_build
def test_reference_run_on_cpu(tmp_path):
    r = subprocess.run([os.path.join(BUILD, "dropin_ref"), str(tmp_path / "ref.bin"), "4"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter_calls=-1" in r.stdout


def _run(exe, path, threads, env=None):
    r = subprocess.run([exe, str(path), str(threads)], capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.fromfile(path, dtype=np.float64), r.stdout


@needs_build
@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 2e-4)])
def test_reference_encoder_with_b200_operator_matches(tmp_path, dtype, tol):
    ref, _ = _run(os.path.join(BUILD, "dropin_ref"), tmp_path / "ref.bin", 4)
    env = dict(os.environ, COTTEN_ADAPTER_DTYPE=dtype)
    gpu, out = _run(os.path.join(BUILD, "dropin_gpu"), tmp_path / "gpu.bin", 4, env)
    calls = int(re.search(r"adapter_calls=(\d+)", out).group(1))
    # 2 layers x 2 heads x 6 sequences, forward and backward
    assert calls >= 2 * 2 * 6 * 2
    # AttentionByteProbe through the drop-in: the adapter's host staging is
    # tracked, so the epoch probe reads > 0 (test_training.cpp:269-272)
    assert int(re.search(r"probe_peak=(\d+)", out).group(1)) > 0
    assert ref.shape == gpu.shape and np.isfinite(gpu).all()
    err = np.abs(gpu - ref).max() / np.abs(ref).max()
    assert err <= tol, f"{dtype}: normwise {err:.3e}"


@needs_build
@pytest.mark.gpu
def test_reference_encoder_at_ml1m_shape_reaches_tcgen05(tmp_path):
    """The reference encoder at the ML-1M shape (N=200, d=64, H=2, |V|=3706,
    dropout 0.1 from the reference's own RNG in both runs): through the
    adapter every head call is a N=200, d_h=32 unit, i.e. the tcgen05
    kernels; logits and every gradient match the pure reference."""
    def run(exe, path, env=None):
        r = subprocess.run([exe, str(path), "8", "bench", "8", "1"], capture_output=True,
                           text=True, timeout=600, env=env)
        assert r.returncode == 0, r.stdout + r.stderr
        return np.fromfile(path, dtype=np.float64), r.stdout
    ref, _ = run(os.path.join(BUILD, "dropin_ref"), tmp_path / "ref.bin")
    gpu, out = run(os.path.join(BUILD, "dropin_gpu"), tmp_path / "gpu.bin",
                   dict(os.environ, COTTEN_ADAPTER_DTYPE="f32"))
    assert int(re.search(r"adapter_calls=(\d+)", out).group(1)) >= 2 * 2 * 8 * 2 * 2
    assert ref.shape == gpu.shape and np.isfinite(gpu).all()
    err = np.abs(gpu - ref).max() / np.abs(ref).max()
    assert err <= 2e-4, f"normwise {err:.3e}"
