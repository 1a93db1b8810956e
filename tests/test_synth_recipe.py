"""The seeded input recipe as generated: mixture
fractions, value ranges and tails of every preset over many batches, and determinism.
-m "not gpu"."""
import numpy as np
import pytest

from paper_2603_25120_b200 import synth


def categories(t, f, x, k):
    video = f > 0
    image = (t > 0) & ~video
    text_only = (t == 0) & (f == 0)
    return image, video, text_only


@pytest.mark.parametrize("k, frac", [(1, dict(image=0.75, video=0.0, text=0.25)),
                                     (2, dict(image=1.0, video=0.0, text=0.0)),
                                     (3, dict(image=0.67, video=0.33, text=0.0)),
                                     (5, dict(image=0.50, video=0.30, text=0.20))])
def test_mixture_fractions(k, frac):
    p = synth.presets()[k]
    feats = [p.features(b) for b in range(12)]
    t, f, x = (np.concatenate([fb[i] for fb in feats]).astype(np.int64) for i in range(3))
    image, video, text_only = categories(t, f, x, k)
    n = len(t)
    tol = 4.0 / np.sqrt(n) + 0.01
    assert abs(image.mean() - frac["image"]) < tol
    assert abs(video.mean() - frac["video"]) < tol
    assert abs(text_only.mean() - frac["text"]) < tol
    assert ((t > 0) & (f > 0)).sum() == 0                     # a sample is image(s) or video
    assert (x >= 8).all()                                     # every sample carries text


def test_ranges_and_tails():
    P = synth.presets()
    t, f, x = (np.concatenate([P[3].features(b)[i] for b in range(20)]).astype(np.int64) for i in range(3))
    v = f[f > 0]
    assert v.min() >= 8 and v.max() <= 512 and (v > 32).mean() > 0.05       # config 3: 15% tail
    t, f, x = (np.concatenate([P[5].features(b)[i] for b in range(8)]).astype(np.int64) for i in range(3))
    assert f.max() <= 768 and t.max() <= 8 * 16 and x.max() <= 32768
    assert np.median(f[f > 0]) >= 16                                          # Pareto(1.1) from 16


def test_deterministic_and_batch_dependent():
    p = synth.presets()[5]
    a, b = p.features(3), p.features(3)
    assert all((u == w).all() for u, w in zip(a, b))
    c = p.features(4)
    assert any((u != w).any() for u, w in zip(a, c))
    assert p.seed(3) == (0xDF100000 + 5, 3)
