"""Mitosis scaling (Sec. 3.5): the oracle's
Fig. 7 walk (N_l = 3, N_u = 6) against the paper's prose and SPEC's worked
examples, invariants, and bit-exact parity of the C++
implementation; InstanceHandler serialization round trip."""
import random

import pytest

from oracle import mitosis as OM


def test_fig7_walk_matches_paper_prose():
    # add until N_u is exceeded -> split off N_l; refill the original; then the new one
    s, seq = [3], []
    for _ in range(10):
        s, a = OM.expand(s, 3, 6)
        seq.append(tuple(s))
    assert seq == [(4,), (5,), (6,), (4, 3), (5, 3), (6, 3), (6, 4), (6, 5), (6, 6), (6, 4, 3)]
    # one macro at 6 + 1 -> {4, 3}
    assert OM.expand([6], 3, 6)[0] == [4, 3]
    # SPEC S:387 / P:597-600: {4, 3} contracting -> the 4-macro shrinks to total N_u, then remove + merge -> {5}
    s = [4, 3]
    s, a = OM.contract(s, 3, 6)
    assert s == [3, 3] and a == ("remove", 0)
    s, a = OM.contract(s, 3, 6)
    assert s == [5] and a[0] == "remove_merge"
    # smallest macro first shrinks to N_l (step 5), then a full macro (step 6)
    assert OM.contract([6, 5], 3, 6)[0] == [6, 4]
    assert OM.contract([6, 3], 3, 6)[0] == [5, 3]


def test_invariants_random_walk():
    rng = random.Random(3)
    for n_l, n_u in [(3, 6), (4, 16), (1, 2), (2, 2)]:
        s, total = [], 0
        for _ in range(400):
            if total == 0 or rng.random() < 0.55:
                s, a = OM.expand(s, n_l, n_u)
                total += 1
            else:
                s, a = OM.contract(s, n_l, n_u)
                total -= 1
            assert sum(s) == total                                   # conservation
            assert all(1 <= v <= n_u for v in s)
            partial = [v for v in s if v < n_u]
            assert len(partial) <= 2 or len(s) <= 2 or n_l == n_u    # "one or two partially filled"


def test_cpp_mitosis_bitexact():
    from paper_2504_18154_b200 import build, macro
    build.build(verbose=False)
    kinds = {"create": 0, "add": 1, "add_split": 2, "remove": 3, "remove_merge": 4, "remove_macro": 5}
    rng = random.Random(9)
    for n_l, n_u in [(3, 6), (4, 16), (1, 3)]:
        s = []
        for _ in range(500):
            expand = not s or rng.random() < 0.5
            ref, ra = (OM.expand if expand else OM.contract)(s, n_l, n_u)
            got, ga = macro.mitosis_step(s, n_l, n_u, expand)
            assert got == ref
            assert ga[0] == kinds[ra[0]] and list(ga[1:1 + len(ra) - 1]) == list(ra[1:])
            s = got


def test_handler_roundtrip_and_version():
    from paper_2504_18154_b200 import build, macro, _lib
    build.build(verbose=False)
    b = macro.handler_to_bytes(42, 3, 2, 1, 9000, "10.0.0.7:5555/gpu3")
    assert b[0] == 1 and len(b) == 31 + len("10.0.0.7:5555/gpu3")
    h = macro.handler_from_bytes(b)
    assert h == dict(actor_id=42, device=3, tp_size=2, tp_rank=1, kv_blocks=9000, address="10.0.0.7:5555/gpu3")
    assert macro.handler_to_bytes(**{**h, "actor_id": 42}) == b
    with pytest.raises(_lib.EcoError) as e:
        macro.handler_from_bytes(bytes([2]) + b[1:])            # unknown wire version
    assert e.value.status == _lib.ERR_UNSUPPORTED
    with pytest.raises(_lib.EcoError):
        macro.handler_from_bytes(b[:-1])                        # truncated
