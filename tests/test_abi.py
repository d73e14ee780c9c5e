"""CPU checks of the boundary: the shared library loads and exports every symbol that
include/kmeans.h declares; the Python binding mirrors those names. No compute calls here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "kmeans.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kmeans_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_core_api():
    names = _declared()
    for core in ("kmeans_create", "kmeans_fit", "kmeans_assign", "kmeans_destroy",
                 "kmeans_last_error", "kmeans_create_dist", "kmeans_cast"):
        assert core in names


def test_library_exports_every_declared_symbol():
    import paper_2407_12208_b200 as mpk
    lib = ctypes.CDLL(mpk.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(mpk.EXPORTS) == _declared()
    for name in _declared():
        assert callable(getattr(mpk, name)), name


def test_library_is_sm100a_only():
    """The .so carries sm_100a SASS (no PTX/CPU fallback path)."""
    import subprocess
    import paper_2407_12208_b200 as mpk
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mpk.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2407_12208_b200 as mpk
    with pytest.raises(mpk.KMeansError) as e:
        mpk.kmeans_create(100, 4, 3, "fp32", "fp16")
    assert e.value.rc in (mpk.KMEANS_ENODEV, mpk.KMEANS_ECUDA)


def test_invalid_arguments_rejected_before_device():
    import paper_2407_12208_b200 as mpk
    bad = [(0, 4, 3, "fp32", "fp16"), (10, 0, 3, "fp32", "fp16"), (10, 4, 11, "fp32", "fp16"),
           (10, 4, 3, "fp16", "fp16"), (10, 4, 3, "fp32", "fp64")]
    for args in bad:
        with pytest.raises(mpk.KMeansError) as e:
            mpk.kmeans_create(*args)
        assert e.value.rc == mpk.KMEANS_EINVAL
    with pytest.raises(mpk.KMeansError):
        mpk.kmeans_create(10, 4, 3, "fp32", "fp16", flags=0x4000)
    assert mpk.kmeans_destroy(None) == 0
