"""The C-ABI library loads and exports every function include/*.h declares
(no compute calls: CPU only)."""

import glob
import os
import re

import pytest

from paper_2404_14044_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\*]+\s+\**(hp_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_binding_table():
    assert _declared() == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.hp_version() == 1
    assert L.hp_last_error() is not None


def test_workspace_size_queries_are_host_only():
    import ctypes
    L = _lib.load()
    nb = _lib.c_size(0)
    assert L.hp_build_workspace_bytes(1000, 64, 48, ctypes.byref(nb)) == 0 and nb.value > 0
    assert L.hp_query_workspace_bytes(4096, 5, 100000, ctypes.byref(nb)) == 0 and nb.value > 0
    p = _lib.SamplerParams(8, 1, 1, 1, 0.02, 0.9, 1e-4, 0.01)
    assert L.hp_sample_workspace_bytes(4096, 100000, 32768, ctypes.byref(p),
                                       ctypes.byref(nb)) == 0 and nb.value > 0


def test_build_rejects_oversized_padded_image_before_any_launch():
    import ctypes
    L = _lib.load()
    cam = _lib.Camera()
    cam.width, cam.height = 70000, 4
    cam.focal_length = cam.pixel_width = cam.pixel_height = 1.0
    L_ = _lib.Layout()
    rc = L.hp_build(None, 0, ctypes.byref(cam), 1, None, None, None, None, None, None, L_, None,
                    None, 0, None)
    assert rc == _lib.HP_EINVAL
    with pytest.raises(ValueError, match="16-bit"):
        _lib.check(rc)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np

    import paper_2404_14044_b200 as hp
    cam = hp.scene_camera(8, 8)
    with pytest.raises(RuntimeError, match="CUDA device"):
        hp.build(hp.PointCloud(np.zeros((3, 3)) + [0, 0, 4]), cam, hp.SearchConfig.for_camera(cam))


def test_head_sort_long_mode_needs_a_ray_list():
    """hp_head_sort's long-head mode (whole > 1024) re-sorts a ray list whose
    head_off the caller spaced for it; without a list it is rejected before
    any launch (hp_head_count spaces head_off for 1024-entry heads)."""
    import ctypes
    L = _lib.load()
    x = ctypes.c_void_p(8)  # never dereferenced: the arguments are rejected first
    args = lambda rays, n, whole: (_lib.Layout(), x, x, 1, x, rays, n, x, 400, whole, x, x, x, x, x,  # noqa: E731
                                   x, x, None, None, 0, None, 0, None)
    assert L.hp_head_sort(*args(None, 0, 2048)) == _lib.HP_EINVAL
    assert L.hp_head_sort(*args(None, 0, 5000)) == _lib.HP_EINVAL
    assert L.hp_head_sort(*args(x, 1, 5000)) == _lib.HP_EINVAL  # past the long heads
