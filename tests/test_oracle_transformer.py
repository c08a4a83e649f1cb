"""Pins of the fp64 transformer oracle (SURVEY 8(c) "What pins each part").

None of these re-type the oracle's formulas: they check closed forms,
invariants, an independent library implementation (torch fp64 SDPA/matmul) and
a brute-force pure-Python loop version on micro shapes.
"""
import math

import numpy as np
import pytest
import torch

from oracle import transformer as T
from synthetic.shapes import ModelShape
from synthetic.weights import make_weights, f32_to_bf16_bits, bf16_bits_to_f32


def test_bf16_rounding_is_rne():
    # 1 + 2^-8 is exactly halfway between bf16 1.0 and 1+2^-7 -> ties to even (1.0)
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 0.0], dtype=np.float32)
    got = bf16_bits_to_f32(f32_to_bf16_bits(x))
    assert got.tolist() == [1.0, 1.0 + 2 ** -6, -2.5, 0.0]


def test_rmsnorm_unit_rms():
    x = np.random.default_rng(0).standard_normal((5, 64)) * 7.0
    y = T.rmsnorm(x, np.ones(64), 0.0)
    np.testing.assert_allclose(np.sqrt(np.mean(y * y, axis=-1)), 1.0, rtol=1e-12)


def test_rope_closed_forms():
    D, theta = 32, 1e4
    rng = np.random.default_rng(1)
    q = rng.standard_normal((1, 1, D))
    c0, s0 = T.rope_cos_sin(np.array([0]), D, theta)
    np.testing.assert_array_equal(T.apply_rope(q, c0, s0), q)           # p = 0 is the identity
    c, s = T.rope_cos_sin(np.array([37]), D, theta)
    np.testing.assert_allclose(np.linalg.norm(T.apply_rope(q, c, s)), np.linalg.norm(q), rtol=1e-12)
    # relative position: q(m).k(n) depends only on m - n
    k = rng.standard_normal((1, 1, D))

    def dot(m, n):
        cm, sm = T.rope_cos_sin(np.array([m]), D, theta)
        cn, sn = T.rope_cos_sin(np.array([n]), D, theta)
        return float(np.sum(T.apply_rope(q, cm, sm) * T.apply_rope(k, cn, sn)))
    assert abs(dot(10, 3) - dot(107, 100)) < 1e-9
    assert abs(dot(10, 3) - dot(3, 10)) > 1e-6   # and is not symmetric in general
    # frequency 0 pair rotates by exactly p radians
    cm, sm = T.rope_cos_sin(np.array([2]), D, theta)
    e = np.zeros((1, 1, D)); e[0, 0, 0] = 1.0
    r = T.apply_rope(e, cm, sm)
    assert abs(r[0, 0, 0] - math.cos(2)) < 1e-15 and abs(r[0, 0, D // 2] - math.sin(2)) < 1e-15


def test_attention_closed_forms():
    rng = np.random.default_rng(2)
    D = 16
    q = rng.standard_normal((1, 2, D)); k = rng.standard_normal((1, 1, D)); v = rng.standard_normal((1, 1, D))
    o = T.attention(q, k, v, np.array([0]), np.array([0]))
    np.testing.assert_allclose(o[0, 0], v[0, 0]); np.testing.assert_allclose(o[0, 1], v[0, 0])
    # identical keys -> uniform weights -> mean of visible values
    kk = np.repeat(rng.standard_normal((1, 1, D)), 5, axis=0)
    vv = rng.standard_normal((5, 1, D))
    qq = rng.standard_normal((5, 1, D))
    o = T.attention(qq, kk, vv, np.arange(5), np.arange(5))
    for i in range(5):
        np.testing.assert_allclose(o[i, 0], vv[:i + 1, 0].mean(axis=0), rtol=1e-12)
    p = T.softmax(rng.standard_normal((4, 9)) * 30)
    np.testing.assert_allclose(p.sum(-1), 1.0, rtol=1e-12)


MICRO = ModelShape("micro", 2, 16, 4, 2, 4, 24, 37, 1e4)


def loop_forward(w, s, tokens):
    """Brute-force pure-Python version of the decoder (micro shapes only):
    every sum written as a loop, independent of the vectorised oracle."""
    H, M, Mkv, D, F = s.hidden, s.n_heads, s.n_kv_heads, s.head_dim, s.ffn_dim
    G = M // Mkv
    n = len(tokens)
    x = [[w["embed"][t][i] for i in range(H)] for t in tokens]

    def norm(row, g):
        ms = sum(a * a for a in row) / len(row)
        r = 1.0 / math.sqrt(ms + s.rms_eps)
        return [row[i] * r * g[i] for i in range(len(row))]

    def mv(W, row):  # W [out][in]
        return [sum(W[o][i] * row[i] for i in range(len(row))) for o in range(len(W))]

    def rope(vec, p):
        out = list(vec)
        for i in range(D // 2):
            ang = p * s.rope_theta ** (-2.0 * i / D)
            a, b = vec[i], vec[i + D // 2]
            out[i] = a * math.cos(ang) - b * math.sin(ang)
            out[i + D // 2] = b * math.cos(ang) + a * math.sin(ang)
        return out

    hidden = [[list(r) for r in x]]
    for l in range(s.n_layers):
        L = w["layers"][l]
        qs, ks, vs = [], [], []
        for t in range(n):
            h = norm(x[t], L["attn_norm"])
            q, k, v = mv(L["wq"], h), mv(L["wk"], h), mv(L["wv"], h)
            qs.append([rope(q[hh * D:(hh + 1) * D], t) for hh in range(M)])
            ks.append([rope(k[g * D:(g + 1) * D], t) for g in range(Mkv)])
            vs.append([v[g * D:(g + 1) * D] for g in range(Mkv)])
        new_x = []
        for t in range(n):
            o = []
            for hh in range(M):
                g = hh // G
                sc = [sum(qs[t][hh][d] * ks[j][g][d] for d in range(D)) / math.sqrt(D) for j in range(t + 1)]
                mx = max(sc)
                e = [math.exp(a - mx) for a in sc]
                z = sum(e)
                o += [sum(e[j] / z * vs[j][g][d] for j in range(t + 1)) for d in range(D)]
            a1 = mv(L["wo"], o)
            x1 = [x[t][i] + a1[i] for i in range(H)]
            h2 = norm(x1, L["ffn_norm"])
            gt, up = mv(L["w_gate"], h2), mv(L["w_up"], h2)
            act = [gt[f] / (1.0 + math.exp(-gt[f])) * up[f] for f in range(F)]
            dn = mv(L["w_down"], act)
            new_x.append([x1[i] + dn[i] for i in range(H)])
        x = new_x
        hidden.append([list(r) for r in x])
    hl = norm(x[-1], w["final_norm"])
    logits = mv(w["lm_head"], hl)
    return hidden, logits


def test_forward_vs_bruteforce_loops():
    w = make_weights(MICRO, seed=3).as_f64()
    m = T.Model(MICRO, w)
    tokens = [5, 0, 36, 17, 17, 2]
    _, out = m.prefill(tokens)
    hid, logits = loop_forward(w, MICRO, tokens)
    for l in range(MICRO.n_layers + 1):
        np.testing.assert_allclose(out.hidden[l], np.array(hid[l]), rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(out.logits, np.array(logits), rtol=1e-11, atol=1e-11)


def torch_forward(w, s, tokens):
    """Independent library implementation: torch fp64 matmul + F.scaled_dot_product_attention."""
    import torch.nn.functional as Fn
    t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64))  # noqa: E731
    n, M, Mkv, D = len(tokens), s.n_heads, s.n_kv_heads, s.head_dim
    x = t(w["embed"])[torch.tensor(tokens)]
    pos = torch.arange(n, dtype=torch.float64)
    inv = 1.0 / (s.rope_theta ** (torch.arange(0, D, 2, dtype=torch.float64) / D))
    ang = torch.outer(pos, inv)
    cos, sin = torch.cat([ang.cos(), ang.cos()], -1), torch.cat([ang.sin(), ang.sin()], -1)

    def rot(z):  # z [heads, n, D]
        z1, z2 = z[..., :D // 2], z[..., D // 2:]
        return z * cos + torch.cat([-z2, z1], -1) * sin

    def rms(z, g):
        return z * torch.rsqrt(z.pow(2).mean(-1, keepdim=True) + s.rms_eps) * t(g)
    hidden = [x]
    for L in w["layers"]:
        h = rms(x, L["attn_norm"])
        q = (h @ t(L["wq"]).T).view(n, M, D).transpose(0, 1)
        k = (h @ t(L["wk"]).T).view(n, Mkv, D).transpose(0, 1)
        v = (h @ t(L["wv"]).T).view(n, Mkv, D).transpose(0, 1)
        o = Fn.scaled_dot_product_attention(rot(q), rot(k), v, is_causal=True, enable_gqa=True)
        x = x + o.transpose(0, 1).reshape(n, M * D) @ t(L["wo"]).T
        h2 = rms(x, L["ffn_norm"])
        x = x + (Fn.silu(h2 @ t(L["w_gate"]).T) * (h2 @ t(L["w_up"]).T)) @ t(L["w_down"]).T
        hidden.append(x)
    logits = rms(x[-1], w["final_norm"]) @ t(w["lm_head"]).T
    return [a.numpy() for a in hidden], logits.numpy()


@pytest.mark.parametrize("name", ["tiny", "tiny-gqa"])
def test_forward_vs_torch_library(name):
    from synthetic.shapes import get_shape
    s = get_shape(name)
    w = make_weights(s, seed=0).as_f64()
    m = T.Model(s, w)
    tokens = list(np.random.default_rng(4).integers(0, s.vocab, 40))
    _, out = m.prefill(tokens)
    hid, logits = torch_forward(w, s, tokens)
    for l in range(s.n_layers + 1):
        np.testing.assert_allclose(out.hidden[l], hid[l], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(out.logits, logits, rtol=1e-9, atol=1e-9)


def test_kv_cached_decode_equals_recompute(tiny_model):
    shape, _, m = tiny_model
    prompt = list(np.random.default_rng(5).integers(0, shape.vocab, 23))
    toks, outs = m.generate(prompt, 5)
    for k in range(1, 5):
        _, full = m.prefill(prompt + toks[:k])
        for l in range(shape.n_layers + 1):
            np.testing.assert_allclose(outs[k].hidden[l][-1], full.hidden[l][-1], rtol=1e-9, atol=1e-9)
        assert full.token == toks[k]


def test_paged_equals_contiguous_bitexact(tiny_model):
    shape, _, m = tiny_model
    rng = np.random.default_rng(6)
    prompt = list(rng.integers(0, shape.vocab, 150))
    nblk = 16
    perm = list(rng.permutation(nblk))
    pool = lambda: [np.full((nblk, shape.n_kv_heads, T.BLOCK_TOKENS, shape.head_dim), np.nan)  # noqa: E731
                    for _ in range(shape.n_layers)]
    paged = T.PagedKV(pool(), pool(), block_table=perm[:4])
    toks_c, outs_c = m.generate(prompt, 4)
    toks_p, outs_p = m.generate(prompt, 4, kv=paged)
    assert toks_c == toks_p
    for a, b in zip(outs_c, outs_p):
        for l in range(shape.n_layers + 1):
            assert np.array_equal(a.hidden[l], b.hidden[l])


def test_tp2_partial_sums_equal_tp1(tiny_model):
    shape, _, m = tiny_model
    tokens = list(np.random.default_rng(7).integers(0, shape.vocab, 30))
    _, out = m.prefill(tokens)
    hid = T.forward_tp(m, tokens, tp=2)
    for l in range(shape.n_layers + 1):
        np.testing.assert_allclose(hid[l], out.hidden[l], rtol=1e-12, atol=1e-12)


def test_greedy_ties_and_nan():
    assert T.greedy(np.array([1.0, 3.0, 3.0, -1.0])) == 1
    with pytest.raises(FloatingPointError):
        T.greedy(np.array([0.0, np.nan]))
    assert T.top2_margin(np.array([0.5, 2.0, 1.25])) == 0.75
