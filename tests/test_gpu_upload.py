"""The native host -> device matrix upload (dpso_upload_matrix: pinned
double buffer, threaded fills): every entry lands, the device padding is
untouched, for the direct (small) and the chunked (> 16 MB) paths, with
contiguous and strided host rows."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1706_04399_b200 import _lib
    from paper_1706_04399_b200.build import build
    build()
    return _lib


@pytest.mark.parametrize("rows,cols,host_pad", [
    (37, 41, 0), (1000, 1000, 0), (3001, 2999, 0), (2500, 2100, 5),
    (1, 5000, 0)])
def test_upload_matrix(lib, rows, cols, host_pad):
    import torch
    rng = np.random.default_rng(rows * 7 + cols)
    host_full = rng.standard_normal((rows, cols + host_pad))
    host = host_full[:, :cols]
    ld = (cols + 7) // 8 * 8
    dev = torch.full((rows, ld), -7.0, dtype=torch.float64, device="cuda")
    lib.check(lib.load().dpso_upload_matrix(
        host_full.ctypes.data, cols + host_pad, rows, cols, dev.data_ptr(),
        ld, torch.cuda.current_stream().cuda_stream))
    got = dev.cpu().numpy()
    assert np.array_equal(got[:, :cols], host)
    assert (got[:, cols:] == -7.0).all()


def test_upload_rejects_bad_arguments(lib):
    import torch
    dev = torch.zeros((4, 8), dtype=torch.float64, device="cuda")
    h = np.zeros((4, 4))
    with pytest.raises(ValueError):
        lib.check(lib.load().dpso_upload_matrix(
            h.ctypes.data, 3, 4, 4, dev.data_ptr(), 8, None))
    with pytest.raises(ValueError):
        lib.check(lib.load().dpso_upload_matrix(
            h.ctypes.data, 4, 4, 4, dev.data_ptr(), 2, None))


def test_upload_to_a_second_device(lib):
    # the chunk events belong to the target stream's device
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    host = np.random.default_rng(5).standard_normal((3000, 3000))
    for d in range(2):
        with torch.cuda.device(d):
            dev = torch.zeros((3000, 3000), dtype=torch.float64,
                              device=f"cuda:{d}")
            lib.check(lib.load().dpso_upload_matrix(
                host.ctypes.data, 3000, 3000, 3000, dev.data_ptr(), 3000,
                torch.cuda.current_stream().cuda_stream))
            assert np.array_equal(dev.cpu().numpy(), host)
