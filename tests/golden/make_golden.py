"""Generate tests/golden/golden.json from the REFERENCE itself.

Runs the reference's own sources (built by oracle/Makefile into
oracle/_ref/libghref.so from /root/reference/proj/src) and records:
  * the SPEC.md worked examples as the reference
    code evaluates them (incl. the two places where code and SPEC differ);
  * encoded frames (proto.cpp:214-274);
  * init_weights / checksum / forward+backward / sgd / easgd outputs on small
    seeded inputs;
  * a short synchronous Downpour run (ref_roles.cpp over InprocHub).
Needs /root/reference at generation time only; the JSON is committed and the
tests read it on any host.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
BENCH = "lstm(5,20,10),softmax(20,3)"
SMALL = "lstm(3,4,5),softmax(4,3)"
DENSE = "dense(2,2,tanh),dense(2,2,identity),softmax(2,3)"


def arr(a):
    return [float(v).hex() for v in np.asarray(a, np.float64).ravel()]


def main():
    O.build()
    R = O.ref()
    g = {"source": "oracle/_ref/libghref.so built from /root/reference/proj/src",
         "float_encoding": "float.hex"}

    # --- sgd_step examples ---
    def sgd(arch, w, v, gr, lr, mu):
        w = np.array(w, np.float64); v = np.array(v, np.float64); gr = np.array(gr, np.float64)
        ver = C.c_uint64(0)
        rc = R.ghr_sgd_step(arch.encode(), O._p(w), O._p(v), O._p(gr), lr, mu, C.byref(ver))
        return rc, w, v, ver.value

    # a 1-parameter-per-tensor architecture does not exist; use the dense net
    # and evaluate the examples on its first element with all others zero.
    P = O.n_params(O.parse_arch(DENSE))
    w = np.zeros(P); w[0] = 1.0
    gr = np.zeros(P); gr[0] = 2.0
    rc, w1, v1, ver = sgd(DENSE, w, np.zeros(P), gr, 0.1, 0.0)
    g["sgd_mu0"] = {"w0": 1.0, "g": 2.0, "lr": 0.1, "w1": w1[0], "version": ver, "rc": rc}
    w = np.zeros(P); w[0] = 1.0
    v = np.zeros(P)
    gr = np.zeros(P); gr[0] = 1.0
    _, w, v, _ = sgd(DENSE, w, v, gr, 0.1, 0.9)
    _, w, v, _ = sgd(DENSE, w, v, gr, 0.1, 0.9)
    g["sgd_two_steps"] = {"w_after": w[0], "expected_spec": 1.0 - 0.1 - 0.19}
    gr = np.zeros(P); gr[3] = np.nan
    rc, w2, _, _ = sgd(DENSE, np.ones(P), np.zeros(P), gr, 0.1, 0.0)
    g["sgd_nan_rc"] = rc
    rc, _, _, _ = sgd(DENSE, np.ones(P), np.zeros(P), np.zeros(P), 0.0, 0.0)
    g["sgd_lr0_rc"] = rc
    rc, _, _, _ = sgd(DENSE, np.ones(P), np.zeros(P), np.zeros(P), 0.1, 1.0)
    g["sgd_mu1_rc"] = rc

    # --- EASGD ---
    w = np.zeros(P); w[0] = 2.0
    c = np.zeros(P)
    R.ghr_easgd_worker_step(DENSE.encode(), O._p(w), O._p(c), O._p(np.zeros(P)), 0.01, 0.5, 1, 0)
    g["easgd_pull_half"] = w[0]
    w = np.zeros(P); w[0] = 8.0
    R.ghr_easgd_worker_step(DENSE.encode(), O._p(w), O._p(c), O._p(np.zeros(P)), 0.01, 0.25, 1, 0)
    a1 = w[0]
    R.ghr_easgd_worker_step(DENSE.encode(), O._p(w), O._p(c), O._p(np.zeros(P)), 0.01, 0.25, 1, 1)
    g["easgd_pull_quarter_twice"] = [a1, w[0]]
    c = np.zeros(P); wk = np.zeros(P); wk[0] = 4.0
    ver = C.c_uint64(0)
    rc = R.ghr_easgd_center_step(DENSE.encode(), O._p(c), O._p(wk), 0.5, C.byref(ver))
    g["easgd_center_mid"] = {"c": c[0], "version": ver.value, "rc": rc}
    rc = R.ghr_easgd_center_step(DENSE.encode(), O._p(np.zeros(P)), O._p(wk), 1.0, C.byref(ver))
    g["easgd_center_alpha1_rc"] = rc  # SPEC.md:164 says c'=w; the code rejects (optim.cpp:32)

    # --- zero weights → uniform probs, loss ln 3 ---
    Pb = O.n_params(O.parse_arch(BENCH))
    x = np.random.default_rng(0).normal(size=(6, 50))
    y = np.array([0, 1, 2, 0, 1, 2], np.int32)
    gz, pz, lz = O.ref_forward_backward(BENCH, np.zeros(Pb), x, y)
    g["zero_weights"] = {"probs": arr(pz), "loss": float(lz).hex(),
                         "bias_grad": arr(gz[-3:])}  # SPEC.md:85 vs code: 1/K - freq

    # --- frames (proto.cpp:214-274) ---
    buf = np.zeros(1 << 16, np.uint8)
    n = C.c_int64()
    R.ghr_encode(0, None, None, 0, 0, 0, O._p(buf, C.c_uint8), len(buf), C.byref(n))
    g["frame_shutdown"] = bytes(buf[: n.value]).hex()
    wb = O.init_weights(O.parse_arch(BENCH), 7)
    R.ghr_encode(1, BENCH.encode(), O._p(wb), 0, 0, 0, O._p(buf, C.c_uint8), len(buf), C.byref(n))
    g["frame_weights_bench_len"] = n.value
    R.ghr_encode(2, BENCH.encode(), O._p(wb), 0, 1000, 0, O._p(buf, C.c_uint8), len(buf),
                 C.byref(n))
    g["frame_gradient_bench_len"] = n.value
    R.ghr_encode(2, BENCH.encode(), O._p(wb), 0, 1000, 1, O._p(buf, C.c_uint8), len(buf),
                 C.byref(n))
    g["frame_gradient_bench_f64_len"] = n.value

    # --- init / checksum / forward+backward on seeded inputs ---
    for name, arch, seed in (("bench", BENCH, 7), ("small", SMALL, 3)):
        w = np.zeros(O.n_params(O.parse_arch(arch)))
        R.ghr_init_weights(arch.encode(), seed, O._p(w))
        cs = C.c_uint64()
        R.ghr_checksum(arch.encode(), O._p(w), C.byref(cs))
        a = O.parse_arch(arch)
        width = O.lib().gho_arch_input_width(C.byref(a))
        xs = np.random.default_rng(seed).normal(size=(9, width)).astype(np.float32).astype(np.float64)
        ys = (np.arange(9) % 3).astype(np.int32)
        gr, pr, lo = O.ref_forward_backward(arch, w, xs, ys)
        g[f"nn_{name}"] = {"arch": arch, "seed": seed, "w": arr(w), "checksum": str(cs.value),
                           "x": arr(xs), "y": ys.tolist(), "grad": arr(gr), "probs": arr(pr),
                           "loss": float(lo).hex()}

    # --- data layer + sync Downpour (c1: 2 workers, B=100) ---
    spec = O.data_spec(10, 500)
    x, y = O.generate(spec)
    g["data_desk"] = {"spec": [10, 500, 10, 5, 3, 5.0, 1234],
                      "x_first_row": arr(x[0]), "x_sum": float(x.sum()).hex(),
                      "label_counts": np.bincount(y).tolist()}
    idx = np.zeros(2500, np.int64); cnt = C.c_int64()
    R.ghr_epoch_indices(C.byref(spec), 2, 1, 3, 99, 1, O._p(idx, C.c_int64), C.byref(cnt))
    g["epoch_indices_w2_k1_e3"] = idx[:40].tolist()
    cfg = O.train_cfg(n_workers=2, batch_size=100, epochs=1, max_updates=20)
    r = O.ref_run_sync(BENCH, spec, x, y, cfg)
    g["sync_c1_20"] = {"cfg": "W=2 B=100 lr=0.01 mu=0.9 seed_w=7 shuffle_seed=99 20 rounds",
                       "w": arr(r.w), "loss": arr(r.loss), "updates": r.stats.updates}
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
