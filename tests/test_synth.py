"""The seeded generator (synth/) is deterministic and follows SURVEY.md §8(d)."""
import numpy as np

import synth


def test_deterministic_and_shapes():
    a = synth.gen_image(37, 53, 5)
    b = synth.gen_image(37, 53, 5)
    assert a.dtype == np.uint8 and a.shape == (37, 53) and a.flags.c_contiguous
    assert np.array_equal(a, b)
    assert not np.array_equal(a, synth.gen_image(37, 53, 6))


def test_noise_level_and_range():
    """Noise sigma matches the config (robust estimate from pixel differences)."""
    for sigma in (10.0, 20.0):
        img = synth.gen_image(512, 512, 1, sigma).astype(np.float64)
        d = np.diff(img, axis=1).ravel()
        mad = np.median(np.abs(d - np.median(d))) / 0.6745 / np.sqrt(2)
        assert abs(mad - sigma) < 0.15 * sigma
        assert img.min() >= 0 and img.max() <= 255


def test_configs_quote_baseline():
    c = synth.CONFIGS
    assert (c["cfg2"].H, c["cfg2"].W) == (1080, 1920)
    assert [c[k].N for k in sorted(c)] == [30, 66, 17, 264, 118]
    assert c["cfg5"].radii == (4, 16, 64)
    assert c["cfg3"].kind == synth.SPATIAL_RAISED_COS
