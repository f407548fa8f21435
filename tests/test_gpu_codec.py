"""GPU wire codec (codec.cu) vs the oracle's restatement of
proto.cpp (itself byte-identical to the reference encoder, tests/test_oracle.py)
and the golden SHUTDOWN frame: frames bit-exact, decode round trips exact,
malformed frames rejected with the reference's DecodeStatus."""
import json
import os

import numpy as np
import pytest

from conftest import BENCH_ARCH

import paper_1712_05878_b200 as g

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
WIDE = "lstm(5,20,10),dense(20,4096,relu),dense(4096,4096,relu),softmax(4096,3)"


@pytest.mark.parametrize("arch_text", [BENCH_ARCH, "lstm(3,4,5),softmax(4,3)",
                                       "lstm(5,20,10),dense(20,64,relu),softmax(64,3)"])
@pytest.mark.parametrize("kind,f64", [(1, False), (2, False), (1, True), (2, True)])
def test_encode_bit_exact_and_round_trip(ctx, oracle, arch_text, kind, f64):
    arch = g.Architecture(ctx, arch_text)
    w = g.init_weights(arch, 11).astype(np.float32)
    fr = g.encode_frame(arch, kind, w, version=123456789012, sample_count=1000, wire_f64=f64)
    a = oracle.parse_arch(arch_text)
    ref = oracle.encode_frame(a, kind, w.astype(np.float64), 123456789012, 1000, int(f64))
    assert fr == ref
    k, w2, ver, cnt, ff = g.decode_frame(arch, fr)
    assert (k, ver, ff) == (kind, 123456789012, f64) and np.array_equal(w2, w)
    assert cnt == (1000 if kind == 2 else 0)


def test_shutdown_and_bench_lengths(ctx):
    arch = g.Architecture(ctx, BENCH_ARCH)
    assert g.encode_frame(arch, g.FRAME_SHUTDOWN).hex() == GOLDEN["frame_shutdown"]
    w = g.init_weights(arch, 7)
    assert len(g.encode_frame(arch, 1, w)) == GOLDEN["frame_weights_bench_len"]
    assert len(g.encode_frame(arch, 2, w, sample_count=1000)) == GOLDEN["frame_gradient_bench_len"]
    assert len(g.encode_frame(arch, 2, w, sample_count=1000, wire_f64=True)) == \
        GOLDEN["frame_gradient_bench_f64_len"]
    assert g.decode_frame(arch, bytes.fromhex(GOLDEN["frame_shutdown"]))[0] == g.FRAME_SHUTDOWN


def test_wide_variant_frame(ctx, oracle):
    """67.5 MB GRADIENT frame of the 16.9 M-parameter wide net."""
    arch = g.Architecture(ctx, WIDE)
    w = (np.random.default_rng(0).normal(size=arch.n_params) * 0.1).astype(np.float32)
    fr = g.encode_frame(arch, 2, w, version=7, sample_count=3)
    assert fr == oracle.encode_frame(oracle.parse_arch(WIDE), 2, w.astype(np.float64), 7, 3, 0)
    assert np.array_equal(g.decode_frame(arch, fr)[1], w)


def test_malformed_frames(ctx, oracle):
    arch = g.Architecture(ctx, BENCH_ARCH)
    a = oracle.parse_arch(BENCH_ARCH)
    w = g.init_weights(arch, 7).astype(np.float32)
    fr = g.encode_frame(arch, 2, w, version=1, sample_count=10)
    bad_version = fr[:4] + b"\x02\x00" + fr[6:]
    bad_type = fr[:6] + b"\x47" + fr[7:]
    plen = int.from_bytes(fr[7:15], "little")
    trailing = fr[:7] + (plen + 1).to_bytes(8, "little") + fr[15:] + b"\x00"  # payload left over
    cases = {1: b"XHUB" + fr[4:], 2: bad_version, 3: fr[:-1], 5: bad_type, 6: trailing}
    # payload length field > 2^40 → length_overflow
    cases[4] = fr[:7] + (1 << 41).to_bytes(8, "little") + fr[15:]
    for status, frame in cases.items():
        with pytest.raises(g.ProtocolError) as e:
            g.decode_frame(arch, frame)
        assert e.value.decode_status == status
        rc, st = oracle.decode_frame(a, frame)[:2]
        assert st == status, (status, st)
    # bytes after the declared payload are not part of the frame (decode reads plen bytes)
    assert g.decode_frame(arch, fr + b"\x00")[0] == 2
    with pytest.raises(g.ShapeError):  # a valid frame of another architecture
        g.decode_frame(arch, g.encode_frame(g.Architecture(ctx, "lstm(3,4,5),softmax(4,3)"), 1,
                                            np.zeros(g.arch_info("lstm(3,4,5),softmax(4,3)")[0])))
    with pytest.raises(g.ConfigError):
        g.encode_frame(arch, 2, w, sample_count=0)


@pytest.mark.parametrize("shift", [4, 8, 12])
@pytest.mark.parametrize("f64", [False, True])
def test_decode_frame_at_unaligned_offsets(ctx, shift, f64):
    """A frame that starts 4/8/12 bytes into a device buffer (not 16-B
    aligned): the unpack kernel's 4-byte staging path, same values."""
    import ctypes as C
    arch = g.Architecture(ctx, "lstm(5,20,10),dense(20,64,relu),softmax(64,3)")
    w = g.init_weights(arch, 5).astype(np.float32)
    fr = g.encode_frame(arch, 2, w, version=9, sample_count=3, wire_f64=f64)
    buf = np.zeros(len(fr) + 16, np.uint8)
    buf[shift:shift + len(fr)] = np.frombuffer(fr, np.uint8)
    d = ctx.upload(buf)
    w2 = ctx.array(arch.n_params)
    kind, ff, st = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    ver, cnt = C.c_uint64(0), C.c_uint64(0)
    g.gradhub.check(ctx.lib.ghc_decode_frame(arch.h, C.c_void_p(d.ptr.value + shift), len(fr), C.byref(kind),
                                             w2.ptr, C.byref(ver), C.byref(cnt), C.byref(ff), C.byref(st)))
    assert (kind.value, ver.value, cnt.value, bool(ff.value)) == (2, 9, 3, f64)
    assert np.array_equal(w2.numpy(), w)
