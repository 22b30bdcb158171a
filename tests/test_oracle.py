"""Pin the oracle before trusting it: every check here compares the oracle with
vectors produced by the reference itself (tests/golden) or with the known answers
hard-coded in the reference's own tests (cited per test). CPU only."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O


# ---------------------------------------------------------------- generators
# test_datagen.py:27-31 GOLDEN splitmix64 outputs
SPLITMIX_GOLDEN = {
    0x0: [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC],
    0x1: [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E, 0x71C18690EE42C90B],
    0xDEADBEEF: [0x4ADFB90F68C9EB9B, 0xDE586A3141A10922, 0x021FBC2F8E1CFC1D, 0x7466CE737BE16790],
}


@pytest.mark.parametrize("seed", sorted(SPLITMIX_GOLDEN))
def test_splitmix_golden(seed):
    g = O.splitmix64(seed)
    assert [next(g) for _ in range(4)] == SPLITMIX_GOLDEN[seed]


def test_small_generated_chunks_match_reference(golden):
    for i, spec in enumerate(golden.meta["gen_small"]):
        px = O.generate(spec["kind"], spec["pixels"], spec["seed"], spec["value"], spec["mean"],
                        spec["sigma"], spec["degeneracy"])
        assert np.array_equal(px, golden[f"gen_small_{i}"]), spec
        assert np.array_equal(O.histogram(px), golden[f"gen_small_{i}_hist"]), spec


def test_big_generated_chunks_match_reference(golden):
    for i, spec in enumerate(golden.meta["gen_big"]):
        px = O.generate(spec["kind"], spec["pixels"], spec["seed"], spec["value"], spec["mean"],
                        spec["sigma"], spec["degeneracy"])
        assert hashlib.sha256(O.pack(px).tobytes()).hexdigest() == spec["sha256"], spec
        assert np.array_equal(O.histogram(px), golden[f"gen_big_{i}_hist"])


def test_mixture_draw_order_matches_pure_python_mirror():
    # test_datagen.py:50-62: Bernoulli first, uniform byte only when needed
    p, v, seed, n = 0.5, 200, 77, 256
    g = O.splitmix64(seed)
    expected = []
    for _ in range(n):
        if (next(g) >> 11) * 2.0 ** -53 < p:
            expected.append(v)
        else:
            expected.append(next(g) & 0xFF)
    assert O.generate("mixture", n, seed, value=v, degeneracy=p).tolist() == expected


def test_normal_matches_pure_python_mirror():
    # test_datagen.py:64-73
    import math

    seed, mean, sigma, n = 13, 127.0, 24.0, 128
    g = O.splitmix64(seed)
    expected = []
    for _ in range(n):
        z = sum((next(g) >> 11) * 2.0 ** -53 for _ in range(12)) - 6.0
        expected.append(min(255, max(0, math.floor(mean + sigma * z + 0.5))))
    assert O.generate("normal", n, seed, mean=mean, sigma=sigma).tolist() == expected


# ---------------------------------------------------------------- histogram + layout
def test_packing_golden():
    # test_core.py:29-32: [1,2,3,4] -> 0x04030201
    assert O.pack(np.array([1, 2, 3, 4], np.uint8)).tolist() == [0x04030201]


def test_hand_count():
    # test_kernels.py:58-61
    h = O.histogram(np.array([1, 1, 2, 0], np.uint8))
    assert h[0] == 1 and h[1] == 2 and h[2] == 1 and h.sum() == 4
    assert O.histogram(np.array([], np.uint8)).sum() == 0


def test_group_ranges_golden(golden):
    # test_kernels.py:274-277 plus reference-generated cases
    assert O.group_ranges(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert O.group_ranges(2, 4) == [(0, 0), (0, 0), (0, 0), (0, 2)]
    for n, g, want in golden.meta["group_ranges"]:
        assert O.group_ranges(n, g) == [tuple(x) for x in want]


def test_naive_and_adaptive_workers_match_reference(golden):
    for i, m in enumerate(golden.meta["slots"]):
        px = golden[f"slots_{i}_pixels"]
        words = O.pack(px)
        off, cnt = golden[f"slots_{i}_offset"], golden[f"slots_{i}_count"]
        gs, gc, S = m["group_size"], m["group_count"], m["total_slots"]
        hist, slots, _ = O.adaptive_histogram(words, off, cnt, S, gs, gc)
        assert np.array_equal(slots, golden[f"slots_{i}_slots"])
        assert np.array_equal(hist, golden[f"slots_{i}_hist"])
        # the numpy simulation (test_kernels.py:28-44) agrees with the arbitration loop
        for got, want in zip(slots, O.simulate_slots(words, off, cnt, S, gs, gc)):
            assert np.array_equal(got, want)
        naive, _ = O.naive_histogram(words, gs, gc)
        assert np.array_equal(naive, O.histogram(px))


def test_lane_touches_match_reference(golden):
    m = golden.meta["touch"]
    words = O.pack(golden["touch_pixels"])
    _, _, tch = O.adaptive_histogram(words, golden["touch_offset"], golden["touch_count"],
                                     int(golden["touch_count"].sum()), m["group_size"], m["group_count"],
                                     touches=True)
    assert np.array_equal(tch, golden["touch_out"])


def test_narrow_slots_match_reference(golden):
    off, cnt = O.uniform_pattern(960)
    _, slots, _ = O.adaptive_histogram(O.pack(golden["narrow_pixels"]), off, cnt, 960, 8, 2, narrow=True)
    assert np.array_equal(slots.astype(np.uint16), golden["narrow_slots"])


def test_narrow_overflow_detectable():
    # test_kernels.py:231-236: 2^20 const pixels over 8 sub-bins -> 131072 per slot
    deg = [0] * 256
    deg[127] = 1_000_000
    off, cnt = O.binning_pattern(deg, 960, 8)
    words = O.pack(np.full(1 << 20, 127, np.uint8))
    hist, _, _ = O.adaptive_histogram(words, off, cnt, 960, 32, 1, narrow=True)
    assert int(hist.sum()) != 1 << 20


def test_eight_subbin_spread():
    # test_kernels.py:140-153: 64 Ki const-127 pixels, cfg(32, 2) -> 8 slots x 8192
    deg = [0] * 256
    deg[127] = 1_000_000
    off, cnt = O.binning_pattern(deg, 960, 8)
    assert cnt[127] == 8
    _, slots, _ = O.adaptive_histogram(O.pack(np.full(1 << 16, 127, np.uint8)), off, cnt, 960, 32, 2)
    comb = slots.sum(axis=0)
    assert (comb[off[127]:off[127] + 8] == (1 << 16) // 8).all()
    assert comb.sum() == 1 << 16


# ---------------------------------------------------------------- pattern
def test_uniform_960_split():
    # test_pattern.py:31-35
    _, cnt = O.uniform_pattern(960)
    assert cnt[:192] == [4] * 192 and cnt[192:] == [3] * 64


def test_degenerate_prior_pattern():
    # test_pattern.py:51-60: count[127] = 8, others 187 x 4 and 68 x 3
    deg = [0] * 256
    deg[127] = 1_000_000
    _, cnt = O.binning_pattern(deg, 960, 8)
    others = cnt[:127] + cnt[128:]
    assert cnt[127] == 8 and others.count(4) == 187 and others.count(3) == 68


def test_patterns_match_reference(golden):
    for i, m in enumerate(golden.meta["patterns"]):
        off, cnt = O.binning_pattern(golden[f"pat_{i}_prior"].tolist(), m["total_slots"], m["cap"])
        assert off == golden[f"pat_{i}_offset"].tolist(), i
        assert cnt == golden[f"pat_{i}_count"].tolist(), i
        assert O.validate_pattern(off, cnt, m["total_slots"], m["cap"]) is None


def test_pattern_text_matches_reference(golden):
    off, cnt = O.uniform_pattern(960)
    text = O.pattern_text(off, cnt)
    assert text == golden.meta["pattern_text_uniform960"]
    lines = text.strip().splitlines()
    assert lines[0] == "0 0 4" and lines[255] == "255 957 3"  # test_pattern.py:151-156


def test_validate_messages_in_order():
    # test_pattern.py:122-147
    off, cnt = O.uniform_pattern(960)
    bad = list(cnt); bad[0] = 0
    assert O.validate_pattern(off, bad, 960, 8) == "count below 1"
    bad = list(cnt); bad[0] = 9
    assert O.validate_pattern(off, bad, 960, 8) == "count above cap"
    bad = list(cnt); bad[0] -= 1; bad[1] += 1
    assert O.validate_pattern(off, bad, 959, 8) == "slot total mismatch"
    boff = list(off); boff[10] += 1
    assert O.validate_pattern(boff, cnt, 960, 8) == "offsets not contiguous"


# ---------------------------------------------------------------- policy
def test_policy_matches_reference(golden):
    for i, m in enumerate(golden.meta["policy"]):
        a, b = golden[f"pol_{i}_a"], golden[f"pol_{i}_b"]
        frac, am, total = O.degeneracy(a)
        assert (frac, am, total) == (m["frac"], m["argmax"], m["total"])
        assert O.select_kernel(frac) == m["kind"]
        if m["divergence"] is not None:
            assert O.divergence(a, b) == m["divergence"]


def test_policy_known_answers():
    # test_policy.py:33-45, :102-115
    a = [0] * 256
    a[127] = 4242
    assert O.degeneracy(a) == (1.0, 127, 4242)
    assert O.degeneracy([10] * 256)[1] == 0
    assert O.degeneracy([0] * 256) == (0.0, 0, 0)
    assert O.select_kernel(0.45) == "adaptive"
    uni = [2] * 256
    mix = [1] * 127 + [257] + [1] * 128
    assert O.divergence(uni, mix) == pytest.approx(255 / 512, abs=1e-12)


# ---------------------------------------------------------------- streaming fold
def _batches(segs, batch_size):
    index = 0
    for spec, n in segs:
        for _ in range(n):
            out = []
            for _ in range(batch_size):
                out.append(O.generate(spec["kind"], spec["pixels"], spec["seed"] ^ index, spec["value"],
                                      spec["mean"], spec["sigma"], spec["degeneracy"]))
                index += 1
            yield out


def test_stream_fold_matches_reference(golden):
    for i, m in enumerate(golden.meta["streams"]):
        r = O.run_sequential(_batches(m["segments"], m["batch_size"]), m["num_iterations"], m["window_size"],
                             m["recompute_pattern_every"])
        assert r["kernel_log"] == m["kernel_log"], i
        assert np.array_equal(np.stack([np.stack(x) for x in r["per_slice"]]), golden[f"stream_{i}_per_slice"])
        assert np.array_equal(r["acc"], golden[f"stream_{i}_acc"])
        assert np.array_equal(r["window"], golden[f"stream_{i}_window"])
        assert np.array_equal(np.stack(r["ring"]), golden[f"stream_{i}_ring"])
        assert r["degeneracy_log"] == golden[f"stream_{i}_deg"].tolist()
        assert r["divergence_log"] == golden[f"stream_{i}_div"].tolist()
        assert r["chunks_seen"] == m["chunks_seen"]


def test_ablation_checksums_match_reference(golden):
    """The genealogy stages' checksums (run_ablation, kernels.py:421-496) on the
    reference's own outputs: seeded chunks, data patterns, 1..5 groups."""
    for i, case in enumerate(golden.meta["ablation"]):
        px = golden[f"ablation_{i}_pixels"]
        off, cnt = O.binning_pattern(O.histogram(px).tolist(), 960, 8)
        got = O.ablation_checksums(px, off, cnt, case["group_count"])
        assert got == case["checksums"], (i, got, case["checksums"])
