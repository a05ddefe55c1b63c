"""hp_host_upload (pageable host -> device through pinned staging, pieces
staged by host threads, DMA per piece): byte-exact for odd sizes, piece
sizes and thread counts; pipeline._h2d on numpy / pageable / pinned inputs."""
import numpy as np
import pytest
import torch

from paper_2404_14044_b200 import pipeline

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes,piece,threads", [(1, 0, 1), (4097, 1024, 3), ((5 << 20) + 13, 1 << 20, 8),
                                                  (3 << 20, 3 << 20, 16), ((9 << 20) + 7, 0, 2)])
def test_host_upload_bytes(nbytes, piece, threads):
    import ctypes
    from paper_2404_14044_b200 import _lib
    lib = _lib.load(require_device=True)
    src = np.random.default_rng(nbytes).integers(0, 256, nbytes, dtype=np.uint8)
    stage = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    out = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    _lib.check(lib.hp_host_upload(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(src.ctypes.data), nbytes,
                                  ctypes.c_void_p(stage.data_ptr()), piece, threads, ctypes.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), src)


def test_h2d_inputs():
    dev = torch.device("cuda")
    rng = np.random.default_rng(0)
    a = rng.random((700_001, 3))
    ints = rng.integers(-5, 5, (400_000, 2))
    for x, dt in ((a, torch.float64), (ints, torch.int64), (a[:, :2], torch.float64),  # non-contiguous view
                  (torch.from_numpy(a), torch.float64), (torch.from_numpy(a).pin_memory(), torch.float64),
                  (a.astype(np.float32), torch.float64), (a[:10], torch.float64)):
        got = pipeline._h2d(x, dev, dt)
        ref = torch.as_tensor(np.asarray(x), dtype=dt)
        torch.cuda.synchronize()
        assert got.shape == ref.shape and got.dtype == dt
        assert torch.equal(got.cpu(), ref)
