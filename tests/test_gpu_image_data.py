"""Image datasets in their distribution formats through the device data path:
a CIFAR-10-format file read by ``load_cifar10`` lives in HBM as its pixel
bytes (``DeviceDataset``, per-batch /255 on the device) and trains the ViT
(NCHW) and ResNet (NHWC) families through ``run_epoch`` — bitwise the same
losses and weights as the host batches of the same file."""
import numpy as np
import pytest
import torch

import paper_2411_12780_b200 as lp

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _cifar(tmp_path, n=96):
    rng = np.random.default_rng(9)
    imgs = rng.integers(0, 256, (n, 3, 32, 32), dtype=np.uint8)
    y = rng.integers(0, 10, n).astype(np.uint8)
    rec = np.concatenate([y[:, None], imgs.reshape(n, -1)], axis=1)
    (tmp_path / "data_batch_1.bin").write_bytes(rec.tobytes())
    return tmp_path / "data_batch_1.bin"


def _flat(m):
    return np.concatenate([p.data.ravel() for p in m.parameters()])


@pytest.mark.parametrize("family", ["vit", "resnet"])
def test_cifar_file_trains_same_on_device_and_host(tmp_path, family):
    path = _cifar(tmp_path)
    layout = "nchw" if family == "vit" else "nhwc"
    ds = lp.load_cifar10(path, layout=layout)
    dd = lp.DeviceDataset(ds)
    assert dd.features.dtype == torch.uint8
    outs = []
    for src in ("host", "device"):
        hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=8, seed=3, precision="bf16")
        if family == "vit":
            spec = lp.VitSpec(image=32, channels=3, patch=4, dim=128, heads=2, mlp=256, depth=2,
                              classes=10)
            mods = lp.build_vit_modules(spec, [1, 1], 1, 2, hyper)
        else:
            mods = lp.build_resnet_modules(lp.ResNetSpec(n=1, image=32, channels=3,
                                                         widths=(16, 32, 64), classes=10),
                                           2, 1, 2, hyper)
        assert mods[0].in_features == ds.dim
        it = lp.batches(ds, 32, True, 4) if src == "host" else dd.batches(32, True, 4)
        met = lp.run_epoch(lp.RunMode.PPLL, mods, it)
        assert met.n_batches == 3
        outs.append((met.loss_history, [_flat(m) for m in mods]))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)
