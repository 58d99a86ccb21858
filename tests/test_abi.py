"""CPU-side checks of the boundary: the C-ABI library loads and exports every
entry point include/synk_cuda.h declares, the Python drop-in imports and
mirrors the reference surface, and host-only pieces (SYNK format, error
classes) behave without a GPU. No device compute here."""

import ctypes
import os
import re
import struct

import numpy as np
import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_1710_04162_b200", "_lib", "libsynk_cuda.so")
HDR = os.path.join(ROOT, "include", "synk_cuda.h")


def declared_symbols():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(synk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("synk_open", "synk_gather_rows", "synk_combine", "synk_weighted_mean", "synk_left_fold",
              "synk_column_stats", "synk_all_reduce", "synk_broadcast", "synk_tree_reduce",
              "synk_optimizer_step", "synk_all_reduce_step", "synk_mlp_loss_grad", "synk_sync"):
        assert s in syms


def test_cabi_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.synk_abi_version.restype = ctypes.c_int
    assert lib.synk_abi_version() == 1


def test_cabi_reports_no_device_cleanly():
    lib = ctypes.CDLL(LIB)
    n = ctypes.c_int(-1)
    rc = lib.synk_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is visible here")
    assert n.value == 0
    assert rc != 0  # no device: an error code, never a silent CPU path
    lib.synk_last_error.restype = ctypes.c_char_p
    assert lib.synk_last_error()


def test_kernels_are_sm100a_only():
    out = os.popen("cuobjdump --list-elf %s 2>/dev/null" % LIB).read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_python_surface_matches_reference(sk):
    # python/synkpar/__init__.py of the reference exports these names
    for name in ("AdamRule", "ArgumentError", "BoundsError", "CapacityError", "CoherenceError", "DTypeError",
                 "Error", "Function", "IoError", "Kernel", "KernelContext", "LifecycleError", "MlpConfig",
                 "MomentumRule", "NumericError", "ParamBlock", "PhaseError", "Pool", "Replicated", "RmsPropRule",
                 "SgdRule", "ShapeError", "SharedInput", "SlicingConflictError", "Trainer", "UseAfterFreeError",
                 "distribute", "load_tensor", "make_function", "make_py_function", "mlp_grad_function",
                 "mlp_grad_kernel", "mlp_init_params", "mlp_make_dataset", "py_kernel", "replicate", "save_tensor"):
        assert hasattr(sk, name), name
    for exc in ("BoundsError", "ShapeError", "DTypeError", "ArgumentError", "LifecycleError", "PhaseError",
                "DeviceError"):
        assert issubclass(getattr(sk, exc), sk.Error)


def test_fork_without_gpu_fails_loudly(sk):
    if sk.device_count() > 0:
        pytest.skip("a GPU is visible here")
    with pytest.raises(sk.DeviceError):
        sk.Pool(workers=2)


@pytest.mark.parametrize("data,hexstr", [
    (np.array([[1, 2], [3, 4]], np.float32),
     "53594e4b01010200020000000000000002000000000000000000803f000000400000404000008040"),
    (np.array([5.5, -2.25]), "53594e4b010201000200000000000000000000000000164000000000000002c0"),
    (np.array(7.0), "53594e4b010200000000000000001c40"),
])
def test_synk_golden_bytes(sk, data, hexstr):
    # test_tensor_io.cpp:28-54, byte strings pinned by the reference
    assert sk.tensor_to_bytes(data) == bytes.fromhex(hexstr)


def test_synk_file_round_trip(sk, tmp_path):
    path = str(tmp_path / "t.synk")
    data = np.linspace(-1, 1, 12).reshape(3, 4)
    sk.save_tensor(path, data)
    blob = open(path, "rb").read()
    assert blob[:4] == b"SYNK" and blob[4] == 1 and blob[5] == 2 and blob[6] == 2
    assert struct.unpack_from("<QQ", blob, 8) == (3, 4)
    np.testing.assert_array_equal(sk.load_tensor(path), data)
    with open(path, "wb") as fh:
        fh.write(b"NOPE" + blob[4:])
    with pytest.raises(sk.IoError):
        sk.load_tensor(path)


def test_synk_bytes_match_reference_writer(sk, oracle):
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("reference module not built here")
    rng = np.random.default_rng(2)
    for arr in (rng.standard_normal((5, 3)).astype(np.float32), rng.standard_normal(7), np.array(3.25)):
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            ref.save_tensor(os.path.join(d, "r.synk"), arr)
            assert open(os.path.join(d, "r.synk"), "rb").read() == sk.tensor_to_bytes(arr)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_synk_streamed_io_and_shared_input_from_file(sk, tmp_path, dtype):
    """SYNK I/O streams: save writes header + payload in place, load_tensor and
    SharedInput.from_file read the payload straight into the destination (the
    pinned store for from_file, shared_input.cpp:75-82). Same bytes, same
    IoError cases (truncated header / extents / payload, bad magic/version/dtype)."""
    path = str(tmp_path / "x.synk")
    data = np.random.default_rng(1).standard_normal((257, 33)).astype(dtype)
    sk.save_tensor(path, data)
    blob = open(path, "rb").read()
    assert blob == sk.tensor_to_bytes(data)
    np.testing.assert_array_equal(sk.load_tensor(path), data)
    arr = sk.SharedInput.from_file(path)
    assert arr.shape == [257, 33] and arr.capacity == data.size
    assert arr.array().tobytes() == data.tobytes()
    big = sk.SharedInput.from_file(path, capacity=data.size * 2)
    assert big.capacity == data.size * 2 and big.array().tobytes() == data.tobytes()
    cases = {
        blob[:5]: "header incomplete",
        blob[:8 + 8]: "extents incomplete",
        blob[:-1]: "payload incomplete",
        b"NOPE" + blob[4:]: "wrong magic",
        blob[:4] + b"\x02" + blob[5:]: "version",
        blob[:5] + b"\x07" + blob[6:]: "dtype code",
    }
    for bad, msg in cases.items():
        with open(path, "wb") as fh:
            fh.write(bad)
        for load in (sk.load_tensor, sk.SharedInput.from_file):
            with pytest.raises(sk.IoError, match=msg):
                load(path)
    with open(path, "wb") as fh:
        fh.write(blob + b"trailing")  # the reference ignores bytes past the payload
    np.testing.assert_array_equal(sk.load_tensor(path), data)


def test_doctest_shim_detects_failures(tmp_path):
    """The doctest-compatible shim used to compile the reference's unit tests
    against this repository really fails on failing checks (CPU only)."""
    import subprocess

    from conftest import ROOT

    src = tmp_path / "t.cpp"
    src.write_text("\n".join([
        "#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN",
        "#include <doctest.h>",
        "#include <stdexcept>",
        'TEST_CASE("ok") { CHECK(1 + 1 == 2); CHECK_THROWS_AS(throw std::runtime_error("x"), std::runtime_error);'
        " CHECK(0.1 + 0.2 == doctest::Approx(0.3)); }",
        'TEST_CASE("bad") { CHECK(1 + 1 == 3); REQUIRE(false); }',
        ""]))
    exe = tmp_path / "t"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-I", os.path.join(ROOT, "tests", "doctest_shim"), str(src), "-o",
                    str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 1
    assert "2 passed" not in out.stdout and "1 passed | 1 failed" in out.stdout
