"""Pins of the accounting oracle against values printed in the paper."""
import json
import os

import pytest

from oracle import accounting as A
from synthetic.shapes import get_shape

GOLD = os.path.join(os.path.dirname(__file__), "golden")
paper = json.load(open(os.path.join(GOLD, "paper_values.json")))
spec = json.load(open(os.path.join(GOLD, "spec_examples.json")))


def test_kv_bytes_per_token_llama30b():
    m = paper["kv_per_token_llama30b"]["model"]
    b = A.kv_bytes_per_token(m["n_layers"], m["n_kv_heads"], m["head_dim"])
    assert b == 1_597_440
    assert round(b / 2 ** 20, 2) == paper["kv_per_token_llama30b"]["mib"]     # P:251 "1.52 MB" (MiB, A21)


def test_kv_totals_printed():
    per = paper["kv_per_token_llama30b"]["mib"]
    g = paper["kv_58p4"]
    assert abs(g["requests"] * g["tokens"] * per / 1000 - g["gb"]) < 0.05     # A21 MiB x decimal mix
    t = paper["kv_178"]
    m = paper["kv_per_token_llama30b"]["model"]
    gib = t["requests"] * t["tokens"] * A.kv_bytes_per_token(m["n_layers"], m["n_kv_heads"], m["head_dim"]) / 2 ** 30
    assert abs(gib - t["gb"]) / t["gb"] < 0.005


@pytest.mark.parametrize("row", paper["table3"]["rows"])
def test_table3_bandwidth(row):
    m = paper["table3"]["models"][row["model"]]
    kv = A.kv_bytes_per_token(m["n_layers"], m["n_kv_heads"], m["head_dim"])
    bw = A.required_kv_bandwidth_gib(row["tokens_per_s"], kv)
    assert abs(bw - row["bandwidth"]) / row["bandwidth"] < 0.002


@pytest.mark.parametrize("case", spec["table2"]["cases"])
def test_table2_worked_examples(case):
    f, _ = A.table2(case["op"], case["phase"], case["B"], case["S"], case["H"], case["M"])
    assert f == case["flops"]


def test_table2_prefill_intensity_exceeds_decode():
    # SPEC S:96 property; Table 2 "Approximate AI" column (BS vs B, S vs 1)
    for op in A.OPS:
        for B, S in [(1, 16), (4, 128), (32, 512)]:
            fp, mp = A.table2(op, "prefill", B, S, 4096, 32)
            fd, md = A.table2(op, "decode", B, S, 4096, 32)
            assert fp / mp >= fd / md


def test_linear_params_match_model_cards():
    # P_lin 8B 6.98e9, 34B 33.2e9, 70B 68.4e9 (public model cards)
    assert abs(A.linear_params(get_shape("8b")) - 6.98e9) / 6.98e9 < 0.002
    assert abs(A.linear_params(get_shape("34b")) - 33.2e9) / 33.2e9 < 0.01
    assert abs(A.linear_params(get_shape("70b")) - 68.4e9) / 68.4e9 < 0.01


def test_kv_bytes_configs():
    assert A.kv_bytes_per_token(32, 8, 128) == 131072      # 8B
    assert A.kv_bytes_per_token(48, 8, 128) == 196608      # 34B (also SPEC S:65)
    assert A.kv_bytes_per_token(80, 4, 128) == 163840      # 70B per TP=2 rank
