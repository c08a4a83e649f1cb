"""CPU checks of the C ABI boundary: the library builds, loads without a GPU and
exports every function include/*.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in ("ecoserve.h", "ecoserve_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(ecoserve_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2504_18154_b200 import build, _lib
    build.build(verbose=False)
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    from paper_2504_18154_b200 import _lib
    names = declared_functions()
    assert len(names) >= 25
    for n in sorted(names):
        assert hasattr(lib, n), f"{n} declared in include/ but not exported"
        assert n in _lib.SIGNATURES, f"{n} has no Python prototype"


def test_size_queries_without_gpu(lib):
    from paper_2504_18154_b200._lib import ModelShape
    s = ModelShape(32, 4096, 32, 8, 128, 14336, 128256, 5e5, 1e-5, 1)
    # 8B: K+V of 32 layers x 8 kv heads x 64 tokens x 128 x bf16 per block = 8 MiB
    assert lib.ecoserve_kv_pool_bytes(ctypes.byref(s), 64, 10) == 10 * 8 * 2 ** 20
    assert lib.ecoserve_kv_pool_bytes(ctypes.byref(s), 32, 10) < 0      # block must be 64
    assert lib.ecoserve_prepared_weight_bytes(ctypes.byref(s)) == 32 * (6144 * 4096 + 2 * 14336 * 4096) * 2
    bad = ModelShape(2, 256, 8, 3, 32, 768, 1024, 1e4, 1e-5, 1)          # Mkv does not divide M
    assert lib.ecoserve_prepared_weight_bytes(ctypes.byref(bad)) < 0


def test_create_rejects_bad_args_without_touching_gpu(lib):
    from paper_2504_18154_b200._lib import ModelShape, KVPool, Weights
    s = ModelShape(2, 256, 8, 8, 32, 768, 1024, 1e4, 1e-5, 1)
    out = ctypes.c_void_p()
    assert lib.ecoserve_instance_create(ctypes.byref(s), None, None, None, 0, 0, None, None, None,
                                        ctypes.byref(out)) == 1
    s2 = ModelShape(2, 256, 8, 8, 32, 768, 1024, 1e4, 1e-5, 2)      # TP=2 needs an NCCL id
    kv = KVPool(64, 4, 1)
    w = Weights(1, 1, 1, ctypes.cast(ctypes.c_void_p(1), ctypes.POINTER(ctypes.c_void_p)))
    assert lib.ecoserve_instance_create(ctypes.byref(s2), ctypes.byref(kv), ctypes.byref(w), ctypes.c_void_p(1), 0, 0,
                                        None, None, None, ctypes.byref(out)) == 1
    s3 = ModelShape(2, 256, 8, 8, 32, 768, 1024, 1e4, 1e-5, 4)      # only TP 1 or 2
    assert lib.ecoserve_prepared_weight_bytes(ctypes.byref(s3)) < 0
    # TP=2 sizes are per rank: half the kv heads, half the QKV/gate-up rows
    assert lib.ecoserve_kv_pool_bytes(ctypes.byref(s2), 64, 1) * 2 == \
        lib.ecoserve_kv_pool_bytes(ctypes.byref(ModelShape(2, 256, 8, 8, 32, 768, 1024, 1e4, 1e-5, 1)), 64, 1)


def test_product_does_not_import_oracle():
    """The product path never imports the oracle (ORACLE header rule)."""
    pkg = os.path.join(ROOT, "paper_2504_18154_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert not re.search(r'#include\s+["<][^">]*oracle', src), f
