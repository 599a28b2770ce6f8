"""CPU checks of the seeded input generator (spgen.gen)."""
import numpy as np

from oracle import ref

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


def test_randn_mode_full_mantissa_rne():
    """"randn" values are the float32 value v * 2^-15 rounded to bf16 to nearest
    even (torch's float32 -> bfloat16 conversion), use the whole 7-bit mantissa,
    and keep the sink / outlier structure."""
    import torch
    w = gen.CONFIGS["C1"].with_(N=600, values="randn")
    vi = gen.gen_K_int(w, 0, 3, 1)
    bits = gen.gen_K(w, 0, 3, 1)
    tb = torch.tensor(vi.astype(np.float32) * np.float32(2.0 ** -15)).to(torch.bfloat16).view(torch.int16)
    np.testing.assert_array_equal(tb.numpy().view(np.uint16), bits)
    assert len(np.unique(bits & 0x7F)) == 128                       # every mantissa pattern occurs
    q = gen.gen_Q(w, 0, 0)
    assert np.array_equal(gen.gen_K(w, 0, 3, 1, 100, 300), bits[100:300])
    v = ref.bf16_to_f64(bits)
    assert 0.9 < v[gen.SINK_TOKENS:, :].std() < 5 and np.abs(v).max() > 10     # outlier channels at +-12.5
    assert np.isfinite(ref.bf16_to_f64(q)).all()


def test_planted_tiers_layout():
    """Ten tiers cut at ceil(j * n_c / 10) (top tier first), chunk 0 in the top
    tier, and the boost only on interior tokens of a boosted chunk."""
    for name in ("C1", "C3", "C4"):
        w = gen.CONFIGS[name].with_(planted=True)
        t = gen.planted_tiers(w, 0)
        n_c = w.n_chunks
        assert t[0] == 9
        cum = np.cumsum(np.bincount(t, minlength=10)[::-1])[:-1]
        assert list(cum) == [(j * n_c + 9) // 10 for j in range(1, 10)]
    w = gen.CONFIGS["C1"].with_(planted=True, L=1, Hkv=1, values="randn")
    t = gen.planted_tiers(w, 0)
    c = int(np.argmax(t[1:] == 5)) + 1
    k1 = gen.gen_K_int(w, 0, 0, 0, c * 32, (c + 1) * 32)
    real = gen.planted_tiers
    try:
        gen.planted_tiers = lambda w_, b_: np.zeros(w_.n_chunks, dtype=np.int64)
        k0 = gen.gen_K_int(w, 0, 0, 0, c * 32, (c + 1) * 32)
    finally:
        gen.planted_tiers = real
    d = k1 - k0
    boost = (gen.PLANT_BASE + gen.PLANT_STEP * 5) * gen.RN_UNIT
    assert not d[:2].any() and not d[30:].any()
    assert set(np.unique(np.abs(d[2:30]))) <= {0, boost} and (np.abs(d[2:30]) == boost).mean() > 0.9
