"""Measured token-budget selection: the calibrate restatement.

host.calibrate (libss_host.so, csrc/host/calibrate.cpp) against
  * the reference's own calibration tests (proj/tests/test_calibrate.cpp:30-106,
    including the bundled configs/calibrate_falcon180b_anchors.json values), and
  * live, the compiled reference (oracle/_ref, servesim::calibrate,
    calibrate.cpp:121-193) on randomized anchor sets: identical fitted constants,
    predictions, zeroed terms and error messages, bit for bit.
"""
import random

import pytest

from paper_2403_02310_b200 import _lib, host

ref = pytest.importorskip("oracle.ref")
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (reference tree absent)")


def decode(count, kv):
    return [host.BatchEntry(i, "decode", 1, kv) for i in range(count)]


def chunk(tokens, prefix=0):
    return [host.BatchEntry(0, "prefill", tokens, prefix)]


def test_falcon_anchor_timings():  # test_calibrate.cpp:30-43
    anchors = [(chunk(4096), 1150.0), (decode(32, 4096), 200.0), (chunk(2048), 575.0), (decode(1, 4096), 132.0)]
    r = host.calibrate(anchors)
    assert abs(r.predicted_ms[0] - 1150.0) / 1150.0 <= 0.10
    assert abs(r.predicted_ms[1] - 200.0) / 200.0 <= 0.10
    assert r.zeroed_terms == ["attn_kv_read_ms"]


def test_round_trip_synthetic_anchors():  # test_calibrate.cpp:45-74
    truth = host.model_preset("falcon180b")
    anchors = [(chunk(n), host.iteration_time(chunk(n), truth)) for n in (1024, 2048, 4096, 6144)]
    anchors += [(decode(bs, 4096), host.iteration_time(decode(bs, 4096), truth)) for bs in (1, 8, 32)]
    anchors.append((chunk(512, 2048), host.iteration_time(chunk(512, 2048), truth)))
    anchors.append((chunk(256), host.iteration_time(chunk(256), truth)))
    r = host.calibrate(anchors)
    assert r.max_relative_error <= 0.01
    assert abs(r.params.per_token_linear_ms - truth.per_token_linear_ms) / truth.per_token_linear_ms <= 0.01
    assert abs(r.params.attn_decode_per_kv_ms - truth.attn_decode_per_kv_ms) / truth.attn_decode_per_kv_ms <= 0.01
    mem = lambda p: p.per_token_linear_ms * p.saturation_tokens  # noqa: E731
    assert abs(mem(r.params) - mem(truth)) / mem(truth) <= 0.01


def test_rejections():  # test_calibrate.cpp:76-106
    with pytest.raises(_lib.CalibrationError):
        host.calibrate([(chunk(4096), 1150.0), (decode(32, 4096), 200.0), (chunk(2048), 575.0)])
    with pytest.raises(_lib.CalibrationError):
        host.calibrate([(chunk(n), 0.254 * n) for n in (1024, 2048, 4096, 8192)])
    with pytest.raises(_lib.CalibrationError, match="under-determined"):
        host.calibrate([(decode(1, 1000), 50.0)] * 4 + [(chunk(1), 50.0)])
    with pytest.raises(_lib.CalibrationError, match="positive"):
        host.calibrate([(chunk(4096), 0.0), (decode(32, 4096), 200.0), (chunk(2048), 575.0), (decode(1, 4096), 1.0)])


def _random_anchor_set(rng):
    anchors = []
    for _ in range(rng.randrange(4, 12)):
        kind = rng.random()
        if kind < 0.35:
            ents = decode(rng.randrange(1, 64), rng.randrange(1, 8192))
        elif kind < 0.7:
            ents = chunk(rng.randrange(1, 6000), rng.choice([0, 0, rng.randrange(0, 8192)]))
        else:
            ents = decode(rng.randrange(1, 32), rng.randrange(1, 8192)) + [
                host.BatchEntry(99, "prefill", rng.randrange(1, 2048), rng.randrange(0, 4096))]
        anchors.append((ents, rng.uniform(1.0, 500.0)))
    return anchors


@needs_ref
def test_live_parity_with_reference():
    rng = random.Random(11)
    n_ok = n_err = 0
    for _ in range(60):
        anchors = _random_anchor_set(rng)
        opts = _lib.CalibOpts(rng.choice([1, 64, 128, 256]), rng.choice([0.0, 0.32, 0.5]), rng.choice([64, 512, 2048]))
        rows, keep = host._anchor_rows(anchors)
        st, rp, rpred, rmax, rmask = ref.calibrate(rows, len(anchors), opts)
        try:
            r = host.calibrate(anchors, opts.tile_size, opts.tile_penalty_frac, opts.max_saturation_tokens)
        except _lib.CalibrationError as e:
            assert st == _lib.SS_CALIBRATION and ref.lib().ref_last_error().decode() in str(e)
            n_err += 1
            continue
        assert st == 0
        for f in ("per_token_linear_ms", "saturation_tokens", "attn_prefill_quad_ms", "attn_kv_read_ms",
                  "attn_decode_per_kv_ms", "fixed_overhead_ms", "tile_size", "tile_penalty_frac"):
            assert getattr(r.params, f) == getattr(rp, f), f
        assert r.predicted_ms == rpred and r.max_relative_error == rmax
        assert r.zeroed_terms == [t for i, t in enumerate(host.CALIBRATION_TERMS) if rmask >> i & 1]
        n_ok += 1
    assert n_ok >= 20 and n_err >= 1
