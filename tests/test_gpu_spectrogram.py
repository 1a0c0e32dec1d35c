"""Spectrogram front end (audio.hpp:121-187) on the device
against an fp64 numpy restatement: sine window, one-sided |FFT|^2, the frame
count rule, the -threshold_db silence filter (order preserved), and the error
types.  Power bins are compared relative to each frame's largest bin (1e-10):
small bins of an FFT carry absolute, not relative, rounding error."""
import numpy as np
import pytest

import paper_1106_4198_b200 as E

pytestmark = pytest.mark.gpu


def ref_stft(x, window, hop):
    n = (x.size - window) // hop + 1
    win = np.sin(np.pi * (np.arange(window) + 0.5) / window)
    frames = np.stack([x[i * hop:i * hop + window] * win for i in range(n)], axis=1)
    spec = np.fft.rfft(frames, axis=0)
    return (spec.real ** 2 + spec.imag ** 2)


@pytest.mark.parametrize("window,hop,n", [(512, 256, 16000), (1024, 256, 20000), (8, 3, 100), (600, 150, 5000),
                                          (4096, 1024, 40000), (2, 1, 7)])
def test_stft_power_matches_fft(window, hop, n):
    rng = np.random.default_rng(window + n)
    t = np.arange(n) / 16000.0
    x = 0.3 * np.sin(2 * np.pi * 440 * t) + 0.05 * rng.standard_normal(n)
    got = E.stft_power(x, window, hop)
    ref = ref_stft(x, window, hop)
    assert got.shape == ref.shape == (window // 2 + 1, (n - window) // hop + 1)
    scale = ref.max(axis=0, keepdims=True)
    assert np.max(np.abs(got - ref) / scale) < 1e-10


def test_stft_errors():
    with pytest.raises(E.EngineError) as e:
        E.stft_power(np.ones(100), 7, 2)
    assert e.value.kind == "UnsupportedFormat"
    with pytest.raises(E.EngineError) as e:
        E.stft_power(np.ones(100), 8, 9)
    assert e.value.kind == "UnsupportedFormat"
    with pytest.raises(E.EngineError) as e:
        E.stft_power(np.ones(100), 512, 256)
    assert e.value.kind == "TooShort"


def test_discard_silence():
    rng = np.random.default_rng(4)
    spec = rng.uniform(0.5, 1.0, size=(33, 500))
    quiet = rng.choice(500, 120, replace=False)
    spec[:, quiet] *= 1e-7  # -70 dB
    spec[:, 17] = 0.0
    keep = E.discard_silence(spec, -60.0)
    power = spec.sum(axis=0)
    expect = np.nonzero(power >= power.max() * 10 ** (-60.0 / 10))[0]
    assert np.array_equal(keep, expect) and keep.size == 500 - 121
    assert np.array_equal(E.discard_silence(spec, -80.0), np.nonzero(power > 0)[0])
    with pytest.raises(E.EngineError) as e:
        E.discard_silence(np.zeros((4, 9)))
    assert e.value.kind == "AllSilent"
    with pytest.raises(E.EngineError) as e:
        E.discard_silence(spec, 1.0)  # a floor above the loudest frame keeps nothing
    assert e.value.kind == "AllSilent"
