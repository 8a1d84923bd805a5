"""The image-dataset readers of the paper's configurations (CIFAR-10/100
binary, SVHN .mat, STL-10 binary): files written here in each distribution
format from known arrays, read back, pixel order / label mapping / error
classes checked.  Host-only (CPU)."""
import numpy as np
import pytest

import paper_2411_12780_b200 as lp


def _chw(n, c, h, w, seed=0):
    return np.random.default_rng(seed).integers(0, 256, (n, c, h, w), dtype=np.uint8)


def test_cifar10_binary_roundtrip(tmp_path):
    imgs = _chw(7, 3, 32, 32)
    y = np.arange(7) % 10
    rec = np.concatenate([y[:, None].astype(np.uint8), imgs.reshape(7, -1)], axis=1)
    (tmp_path / "a.bin").write_bytes(rec[:4].tobytes())
    (tmp_path / "b.bin").write_bytes(rec[4:].tobytes())
    ds = lp.load_cifar10([tmp_path / "a.bin", tmp_path / "b.bin"])
    assert ds.n == 7 and ds.dim == 3072 and ds.num_classes == 10 and ds.shape == (3, 32, 32)
    np.testing.assert_array_equal(ds.labels, y)
    np.testing.assert_array_equal(ds.pixels, imgs.reshape(7, -1))               # NCHW
    np.testing.assert_array_equal(ds.features, (imgs.reshape(7, -1) / 255.0).astype(np.float32))
    nhwc = lp.load_cifar10(tmp_path / "a.bin", layout="nhwc")
    np.testing.assert_array_equal(nhwc.pixels.reshape(4, 32, 32, 3), imgs[:4].transpose(0, 2, 3, 1))
    # CIFAR-100: coarse + fine label bytes, the fine one is used
    rec100 = np.concatenate([np.full((7, 1), 3, np.uint8), (y + 50)[:, None].astype(np.uint8),
                             imgs.reshape(7, -1)], axis=1)
    (tmp_path / "c.bin").write_bytes(rec100.tobytes())
    ds100 = lp.load_cifar10(tmp_path / "c.bin", cifar100=True)
    np.testing.assert_array_equal(ds100.labels, y + 50)
    assert ds100.num_classes == 100


def test_cifar10_errors(tmp_path):
    (tmp_path / "t.bin").write_bytes(b"\x00" * 3000)
    with pytest.raises(lp.TruncatedFile):
        lp.load_cifar10(tmp_path / "t.bin")
    with pytest.raises(lp.InvalidArg):
        (tmp_path / "ok.bin").write_bytes(b"\x01" + b"\x00" * 3072)
        lp.load_cifar10(tmp_path / "ok.bin", layout="hwcn")
    (tmp_path / "bad.bin").write_bytes(b"\x0c" + b"\x00" * 3072)          # label 12
    with pytest.raises(lp.InvalidArg):
        lp.load_cifar10(tmp_path / "bad.bin")


def test_svhn_mat_roundtrip(tmp_path):
    from scipy.io import savemat
    imgs = _chw(5, 3, 32, 32, seed=1)
    y = np.array([10, 1, 2, 9, 10])                     # digit 0 is stored as 10
    savemat(tmp_path / "s.mat", {"X": imgs.transpose(2, 3, 1, 0), "y": y[:, None]})
    ds = lp.load_svhn(tmp_path / "s.mat")
    np.testing.assert_array_equal(ds.labels, [0, 1, 2, 9, 0])
    np.testing.assert_array_equal(ds.pixels, imgs.reshape(5, -1))
    nhwc = lp.load_svhn(tmp_path / "s.mat", layout="nhwc")
    np.testing.assert_array_equal(nhwc.pixels.reshape(5, 32, 32, 3), imgs.transpose(0, 2, 3, 1))
    savemat(tmp_path / "m.mat", {"X": imgs.transpose(2, 3, 1, 0), "y": y[:4, None]})
    with pytest.raises(lp.CountMismatch):
        lp.load_svhn(tmp_path / "m.mat")


def test_stl10_binary_roundtrip(tmp_path):
    imgs = _chw(3, 3, 96, 96, seed=2)
    # STL-10 stores every channel plane column-major
    (tmp_path / "x.bin").write_bytes(np.ascontiguousarray(imgs.transpose(0, 1, 3, 2)).tobytes())
    (tmp_path / "y.bin").write_bytes(np.array([1, 10, 5], np.uint8).tobytes())
    ds = lp.load_stl10(tmp_path / "x.bin", tmp_path / "y.bin")
    np.testing.assert_array_equal(ds.labels, [0, 9, 4])
    np.testing.assert_array_equal(ds.pixels, imgs.reshape(3, -1))
    assert ds.shape == (3, 96, 96)
    (tmp_path / "y2.bin").write_bytes(np.array([1, 2], np.uint8).tobytes())
    with pytest.raises(lp.CountMismatch):
        lp.load_stl10(tmp_path / "x.bin", tmp_path / "y2.bin")
    (tmp_path / "x2.bin").write_bytes(b"\x00" * 100)
    with pytest.raises(lp.TruncatedFile):
        lp.load_stl10(tmp_path / "x2.bin", tmp_path / "y.bin")


def test_image_dataset_batches_follow_reference_order(tmp_path):
    imgs = _chw(10, 3, 32, 32, seed=3)
    rec = np.concatenate([(np.arange(10) % 10)[:, None].astype(np.uint8), imgs.reshape(10, -1)], 1)
    (tmp_path / "a.bin").write_bytes(rec.tobytes())
    ds = lp.load_cifar10(tmp_path / "a.bin")
    got = list(lp.batches(ds, 4, shuffle=True, seed=5))
    order = np.random.default_rng(5).permutation(10)
    np.testing.assert_array_equal(np.concatenate([y for _, y in got]), ds.labels[order])
    assert [x.shape[0] for x, _ in got] == [4, 4, 2]
