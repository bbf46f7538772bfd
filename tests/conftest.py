import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size case")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def split_corpus(shapes, flat_pixels, flat_words=None):
    """Cut the concatenated fixture arrays back into per-image pieces."""
    pix, words = [], []
    po = wo = 0
    for h, w in shapes:
        h, w = int(h), int(w)
        pix.append(flat_pixels[po:po + h * w].reshape(h, w))
        po += h * w
        if flat_words is not None:
            wp = -(-w // 64)
            words.append(flat_words[wo:wo + h * wp].reshape(h, wp))
            wo += h * wp
    return pix, words


def exhaustive_images(n: int) -> np.ndarray:
    total = 1 << (n * n)
    idx = np.arange(total, dtype=np.int64)
    sh = np.arange(n * n, dtype=np.int64)
    return ((idx[:, None] >> sh[None, :]) & 1).astype(np.uint8).reshape(total, n, n)


def encode_bits(arr: np.ndarray) -> np.ndarray:
    """[K, n, n] uint8 bits -> uint16 with pixel (x, y) at bit y*n + x (make_golden encoding)."""
    k = arr.shape[0]
    flat = arr.reshape(k, -1).astype(np.int64)
    weights = (1 << np.arange(flat.shape[1], dtype=np.int64))
    return (flat * weights).sum(1).astype(np.uint16)


@pytest.fixture(autouse=True)
def _dispatch_knobs(monkeypatch):
    """The library reads its BITEDGE_* dispatch knobs once per process: re-read
    them at the start of every test and after every monkeypatch.setenv/delenv
    (the knob-sweeping tests set them inside the test body)."""
    import importlib

    def reload():
        try:
            capi = importlib.import_module("paper_1401_5245_b200._capi")
            if capi._lib is not None:
                capi.reload_knobs()
        except Exception:
            pass

    setenv, delenv = monkeypatch.setenv, monkeypatch.delenv

    def setenv_(name, value, prepend=None):
        setenv(name, value, prepend)
        reload()

    def delenv_(name, raising=True):
        delenv(name, raising)
        reload()

    monkeypatch.setenv, monkeypatch.delenv = setenv_, delenv_
    reload()
    yield


@pytest.fixture(scope="session")
def cuda_dev():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1401_5245_b200 import _capi

    _capi.load()
    return torch.device("cuda", 0)
