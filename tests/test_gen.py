"""CPU checks of the seeded input generator (spgen.gen)."""
import numpy as np

from spgen import gen


def test_values_exact_in_bf16_and_deterministic():
    w = gen.CONFIGS["C1"].with_(N=512)
    k = gen.gen_K_int(w, 0, 3, 5)
    assert k.shape == (512, 128) and np.abs(k).max() <= 255
    bits = gen.gen_K(w, 0, 3, 5)
    f = (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)
    np.testing.assert_array_equal(f.astype(np.float64) * 64.0, k.astype(np.float64))
    np.testing.assert_array_equal(bits, gen.gen_K(w, 0, 3, 5))
    q = gen.gen_Q_int(w, 0, 7)
    assert q.shape == (8, 32, 128) and np.abs(q).max() <= 255


def test_slices_are_consistent():
    """Any token range regenerates identically (sequence shards, sampled checks)."""
    w = gen.CONFIGS["C1"].with_(N=1000)
    full = gen.gen_K(w, 0, 1, 2)
    np.testing.assert_array_equal(gen.gen_K(w, 0, 1, 2, 123, 777), full[123:777])
    tok = gen.gen_tokens(w, 0)
    np.testing.assert_array_equal(gen.gen_tokens(w, 0, 10, 20), tok[10:20])
    assert tok.min() >= 0 and tok.max() < gen.VOCAB


def test_structure_present():
    w = gen.CONFIGS["C1"]
    spans = gen.needle_spans(w, 0)
    assert 1 <= len(spans) <= 4
    for s, e in spans:
        assert 16 <= e - s <= 64 and 0 <= s < e <= w.N
    assert gen.needle_spans(gen.CONFIGS["C0"], 0) == []
    k = gen.gen_K_int(w, 0, 0, 0, 0, 8)
    u = gen._usign(w, 0, 0, 0, np.arange(w.d, dtype=np.uint64))
    # sink tokens lean along u
    assert (k[:4] * u[None, :]).sum() > (k[4:8] * u[None, :]).sum()


def test_seeds_differ():
    a = gen.gen_K(gen.CONFIGS["C0"], 0, 0, 0)
    b = gen.gen_K(gen.CONFIGS["C0"].with_(seed=1), 0, 0, 0)
    assert (a != b).mean() > 0.5
