"""CPU: the C-ABI library loads, exports every symbol include/ghc.h declares,
and its host-side layers (architecture grammar, init_weights, data layer) are
bit-identical to the oracle.  No compute calls (no GPU here)."""
import os
import re

import numpy as np
import pytest

from conftest import BENCH_ARCH, ROOT

import paper_1712_05878_b200 as g
from paper_1712_05878_b200 import _lib


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ghc.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(ghc_[a-z0-9_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 40
    for n in names:
        assert hasattr(lib, n), n
    assert set(n for n, _, _ in _lib.SIGNATURES) == set(names)


def test_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    import ctypes as C
    n = C.c_int()
    if _lib.load().ghc_device_count(C.byref(n)) == 0 and n.value > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(g.CudaError):
        g.Context(0)


@pytest.mark.parametrize("text,ok", [
    (BENCH_ARCH, True), ("dense(2,3,tanh),softmax(3,3)", True),
    ("lstm(5,20,10), dense(20,8,relu) ,softmax(8,3)", True),
    ("softmax(3,3),dense(3,3,tanh)", False), ("dense(2,3,tanh),softmax(4,3)", False),
    ("dense(2,3,tanh),lstm(3,2,2),softmax(2,3)", False), ("dense(2,3,sigmoid),softmax(3,3)", False),
    ("lstm(5,20,10),softmax(20,3),", False), ("", False), ("dense(2,3,tanh)", False)])
def test_architecture_grammar(oracle, text, ok):
    if ok:
        n, wdt, k = g.arch_info(text)
        a = oracle.parse_arch(text)
        assert n == oracle.n_params(a) and k == a.b[a.n_layers - 1]
    else:
        with pytest.raises(g.ConfigError):
            g.arch_info(text)


@pytest.mark.parametrize("text,seed", [(BENCH_ARCH, 7), ("dense(50,9,relu),softmax(9,3)", 3),
                                       ("lstm(3,4,5),softmax(4,3)", 123)])
def test_init_weights_bitexact(oracle, text, seed):
    assert np.array_equal(g.init_weights(text, seed),
                          oracle.init_weights(oracle.parse_arch(text), seed))


def test_data_generate_bitexact(oracle):
    spec = g.data_spec(6, 37, delta=3.0, seed=99)
    x, y = g.generate(spec)
    xo, yo = oracle.generate(oracle.data_spec(6, 37, delta=3.0, seed=99))
    assert np.array_equal(x.astype(np.float64), xo) and np.array_equal(y, yo)
    xs, ys = g.generate(spec, 2, 3)
    assert np.array_equal(xs, x[2 * 37:5 * 37]) and np.array_equal(ys, y[2 * 37:5 * 37])


@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_sharding_and_indices_bitexact(oracle, W):
    spec = g.data_spec(17, 23)
    so = oracle.data_spec(17, 23)
    for k in range(W):
        for e in range(3):
            for sh in (True, False):
                assert np.array_equal(g.epoch_indices(spec, W, k, e, 4242, sh),
                                      oracle.epoch_indices(so, W, k, e, 4242, sh))


def test_batches_short_final(oracle):
    spec = g.data_spec(3, 10)
    bs = g.batches(spec, 1, 0, 7, 2, 1)
    assert [len(b) for b in bs] == [7, 7, 7, 7, 2] * 2
    assert sorted(np.concatenate(bs[:5]).tolist()) == list(range(30))
