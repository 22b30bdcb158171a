"""Host-side product logic on the CPU: value types, the native pattern/policy
control plane and the native host generators, checked against the oracle and the
reference-generated golden vectors. No GPU calls."""
import io

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200.datagen import batch_stream, chunk_stream, derived_spec, load_raw_file, schedule_stream


# ---------------------------------------------------------------- core (core.py)
def test_packing_and_unpacking():
    c = hs.pack_pixels([1, 2, 3, 4])
    assert c.words.tolist() == [0x04030201] and c.pixel_count == 4
    assert hs.pack_pixels([7] * 8).words.tolist() == [0x07070707] * 2
    assert hs.unpack_word(0xFF0000FF) == (255, 0, 0, 255)
    assert hs.pack_pixels([]).pixel_count == 0
    with pytest.raises(hs.LengthNotMultipleOfFour):
        hs.pack_pixels([1, 2, 3])
    with pytest.raises(hs.PixelValueOutOfRange):
        hs.pack_pixels([0, 1, 2, 256])
    with pytest.raises(hs.PixelValueOutOfRange):
        hs.pack_pixels([-1, 1, 2, 3])


@given(st.lists(st.integers(0, 255), max_size=256).filter(lambda p: len(p) % 4 == 0))
def test_round_trip(pixels):
    c = hs.pack_pixels(pixels)
    assert hs.unpack_chunk(c).tolist() == pixels
    for i, w in enumerate(c.words):
        assert list(hs.unpack_word(int(w))) == pixels[4 * i:4 * i + 4]


def test_immutability():
    c = hs.pack_pixels([1, 2, 3, 4])
    with pytest.raises(ValueError):
        c.words[0] = 5
    with pytest.raises(AttributeError):
        c.words = np.zeros(1, np.uint32)
    h = hs.zero_histogram()
    with pytest.raises(ValueError):
        h.counts[0] = 3
    with pytest.raises(ValueError):
        hs.Histogram256(np.zeros(255, np.uint64))


def test_merge_semantics():
    a = np.zeros(256, np.uint64); a[1] = 2
    b = np.zeros(256, np.uint64); b[1] = 3; b[2] = 1
    m = hs.merge(hs.Histogram256(a), hs.Histogram256(b))
    assert m.counts[1] == 5 and m.counts[2] == 1
    big = np.zeros(256, np.uint64); big[0] = (1 << 64) - 1
    one = np.zeros(256, np.uint64); one[0] = 1
    with pytest.raises(hs.CountOverflow):
        hs.merge(hs.Histogram256(big), hs.Histogram256(one))
    assert hs.merge_all([]) == hs.zero_histogram()


def test_group_ranges_matches_oracle(golden, oracle):
    for n, g, want in golden.meta["group_ranges"]:
        assert hs.group_ranges(n, g) == [tuple(x) for x in want] == oracle.group_ranges(n, g)


# ---------------------------------------------------------------- pattern (native control plane)
def test_patterns_bit_identical_to_reference(golden):
    for i, m in enumerate(golden.meta["patterns"]):
        p = hs.compute_binning_pattern(hs.Histogram256(golden[f"pat_{i}_prior"]), m["total_slots"], m["cap"])
        assert np.array_equal(p.offset, golden[f"pat_{i}_offset"]), i
        assert np.array_equal(p.count, golden[f"pat_{i}_count"]), i


@settings(max_examples=300, deadline=None)
@given(seed=st.integers(0, 2**32 - 1), slots=st.integers(256, 2048), cap=st.integers(1, 8), shape=st.integers(0, 4))
def test_patterns_match_oracle(oracle, seed, slots, cap, shape):
    slots = min(slots, 256 * cap)
    rng = np.random.default_rng(seed)
    if shape == 0:
        c = rng.integers(0, 1 << 20, 256)
    elif shape == 1:
        c = np.zeros(256, np.int64); c[rng.integers(0, 256)] = rng.integers(1, 1 << 40)
    elif shape == 2:
        c = np.zeros(256, np.int64)
    elif shape == 3:
        c = rng.zipf(1.7, 256)
    else:
        c = np.full(256, int(rng.integers(1, 5000)), np.int64); c[:: int(rng.integers(2, 9))] += 1
    prior = c.astype(np.uint64)
    p = hs.compute_binning_pattern(hs.Histogram256(prior), slots, cap)
    off, cnt = oracle.binning_pattern(prior.tolist(), slots, cap)
    assert p.offset.tolist() == off and p.count.tolist() == cnt
    hs.validate_pattern(p)


def test_uniform_and_degenerate_patterns():
    p = hs.uniform_pattern(960)
    assert (p.count[:192] == 4).all() and (p.count[192:] == 3).all()
    assert hs.compute_binning_pattern(hs.zero_histogram(), 960) == p
    assert (hs.uniform_pattern(2048, cap=8).count == 8).all()
    d = np.zeros(256, np.uint64); d[127] = 1_000_000
    q = hs.compute_binning_pattern(hs.Histogram256(d), 960, 8)
    assert q.count[127] == 8 and q.hot_bin == 127
    for bad in (255, 100, 2049, 10_000):
        with pytest.raises(hs.SlotCountOutOfRange):
            hs.uniform_pattern(bad, cap=8)
        with pytest.raises(hs.SlotCountOutOfRange):
            hs.compute_binning_pattern(hs.zero_histogram(), bad, 8)


def test_validate_pattern_messages():
    base = hs.uniform_pattern(960)

    def with_count(mut, total=960):
        c = base.count.copy(); mut(c)
        return hs.BinningPattern(base.offset, c, total, 8)

    with pytest.raises(hs.InvalidPattern, match="count below 1"):
        hs.validate_pattern(with_count(lambda c: c.__setitem__(0, 0)))
    with pytest.raises(hs.InvalidPattern, match="count above cap"):
        hs.validate_pattern(with_count(lambda c: c.__setitem__(0, 9)))

    def swap(c):
        c[0] -= 1; c[1] += 1
    with pytest.raises(hs.InvalidPattern, match="slot total mismatch"):
        hs.validate_pattern(with_count(swap, 959))
    off = base.offset.copy(); off[10] += 1
    with pytest.raises(hs.InvalidPattern, match="offsets not contiguous"):
        hs.validate_pattern(hs.BinningPattern(off, base.count, 960, 8))
    with pytest.raises(hs.InvalidPattern, match="256 entries"):
        hs.validate_pattern(hs.BinningPattern(base.offset[:10], base.count[:10], 960, 8))


def test_pattern_text(golden):
    assert hs.pattern_to_text(hs.uniform_pattern(960)) == golden.meta["pattern_text_uniform960"]
    rng = np.random.default_rng(23)
    p = hs.compute_binning_pattern(hs.Histogram256(rng.integers(0, 999, 256).astype(np.uint64)), 960)
    assert hs.pattern_from_text(hs.pattern_to_text(p)) == p


# ---------------------------------------------------------------- policy
def test_policy_matches_reference(golden):
    for i, m in enumerate(golden.meta["policy"]):
        a, b = hs.Histogram256(golden[f"pol_{i}_a"]), hs.Histogram256(golden[f"pol_{i}_b"])
        d = hs.degeneracy(a)
        assert (d.max_bin_fraction, d.argmax_bin, d.total) == (m["frac"], m["argmax"], m["total"])
        assert hs.select_kernel(d, hs.SwitchPolicy()).value == m["kind"]
        if m["divergence"] is not None:
            assert hs.divergence(a, b) == m["divergence"]


def test_native_divergence_is_numpy_pairwise(oracle):
    """hs_divergence (native, numpy's pairwise summation order) against the oracle's numpy
    restatement of policy.py:56-64, bit for bit, over count scales from 1 to 2**62."""
    rng = np.random.default_rng(64)
    for trial in range(4000):
        scale_a, scale_b = 2 ** int(rng.integers(1, 62)), 2 ** int(rng.integers(1, 62))
        a = rng.integers(0, scale_a, 256, dtype=np.uint64)
        b = rng.integers(0, scale_b, 256, dtype=np.uint64)
        if trial % 5 == 0:
            a[rng.random(256) < 0.9] = 0
        if int(a.sum(dtype=object)) == 0 or int(b.sum(dtype=object)) == 0 or a.sum(dtype=object) >= 2**64:
            continue
        if b.sum(dtype=object) >= 2**64:
            continue
        want = oracle.divergence(a, b)
        assert hs.divergence(hs.Histogram256(a), hs.Histogram256(b)) == want, trial


def test_policy_edges():
    assert hs.degeneracy(hs.zero_histogram()) == hs.DegeneracyReport(0.0, 0, 0)
    assert hs.select_kernel(hs.DegeneracyReport(0.45, 5, 10), hs.SwitchPolicy(0.45)) is hs.KernelKind.ADAPTIVE
    assert hs.select_kernel(hs.DegeneracyReport(1 / 256, 0, 10), hs.SwitchPolicy()) is hs.KernelKind.NAIVE
    for bad in (0.0, 1.0):
        with pytest.raises(ValueError):
            hs.SwitchPolicy(bad)
    with pytest.raises(hs.EmptyHistogram):
        hs.divergence(hs.zero_histogram(), hs.zero_histogram())


@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(0, 2**40), min_size=256, max_size=256))
def test_degeneracy_matches_oracle(oracle, counts):
    d = hs.degeneracy(hs.Histogram256(np.array(counts, np.uint64)))
    assert (d.max_bin_fraction, d.argmax_bin, d.total) == oracle.degeneracy(counts)


# ---------------------------------------------------------------- generators (native host)
def test_generators_match_reference(golden):
    for i, s in enumerate(golden.meta["gen_small"]):
        spec = hs.SourceSpec(s["kind"], s["pixels"], s["seed"], s["value"], s["mean"], s["sigma"], s["degeneracy"])
        assert np.array_equal(hs.unpack_chunk(hs.generate(spec)), golden[f"gen_small_{i}"]), s


def test_big_generators_match_reference(golden):
    import hashlib

    for s in golden.meta["gen_big"]:
        spec = hs.SourceSpec(s["kind"], s["pixels"], s["seed"], s["value"], s["mean"], s["sigma"], s["degeneracy"])
        assert hashlib.sha256(hs.generate(spec).words.tobytes()).hexdigest() == s["sha256"]


@pytest.mark.parametrize("kind", ["uniform", "normal", "mixture", "sequential", "constant"])
def test_multithreaded_host_generator_matches_oracle(oracle, kind):
    spec = hs.SourceSpec(kind, (1 << 21) + 12, seed=0xC0FFEE, value=9, mean=120.5, sigma=17.0, degeneracy=0.3)
    got = hs.unpack_chunk(hs.generate(spec))
    want = oracle.generate(kind, spec.pixels, spec.seed, spec.value, spec.mean, spec.sigma, spec.degeneracy)
    assert np.array_equal(got, want)


def test_spec_validation_and_streams(tmp_path):
    for bad in (hs.SourceSpec("uniform", 10, 0), hs.SourceSpec("mixture", 8, 0, degeneracy=1.5),
                hs.SourceSpec("normal", 8, 0, sigma=0.0), hs.SourceSpec("constant", 8, 0, value=300),
                hs.SourceSpec("nope", 8, 0), hs.SourceSpec("file", 0, 0, path=None)):
        with pytest.raises(hs.SpecInvalid):
            hs.generate(bad)
    assert derived_spec(hs.SourceSpec("uniform", 8, seed=0b1010), 0b0110).seed == 0b1100
    spec = hs.SourceSpec("uniform", 16, seed=7)
    flat = [c for b in batch_stream(spec, 3, 2) for c in b]
    assert all(c == hs.generate(derived_spec(spec, i)) for i, c in enumerate(flat))
    assert list(chunk_stream(spec, 2)) == [hs.generate(derived_spec(spec, i)) for i in range(2)]
    a, b = hs.SourceSpec("uniform", 16, seed=1), hs.SourceSpec("constant", 16, seed=1, value=127)
    sched = list(schedule_stream([(a, 2), (b, 1)]))
    assert sched[2][0] == hs.generate(derived_spec(b, 2))
    p = tmp_path / "raw.bin"
    p.write_bytes(bytes(range(10)))
    assert load_raw_file(p).pixel_count == 8
    with pytest.raises(hs.FileUnreadable):
        load_raw_file(tmp_path / "missing.bin")


def test_pipeline_config_validation():
    for kw in (dict(num_iterations=0), dict(num_iterations=1, chunk_pixels=6), dict(num_iterations=1, batch_size=0),
               dict(num_iterations=1, recompute_pattern_every=0), dict(num_iterations=1, window_size=0)):
        with pytest.raises(ValueError):
            hs.PipelineConfig(**kw)
    with pytest.raises(ValueError):
        hs.WorkerGroupConfig(0, 1)
    with pytest.raises(ValueError):
        hs.WindowState(0)


def test_window_and_accumulator_fold():
    rng = np.random.default_rng(5)
    hists = [hs.Histogram256(rng.integers(0, 10_000, 256).astype(np.uint64)) for _ in range(300)]
    win, acc = hs.WindowState(32), hs.AccumulatorState()
    for h in hists:
        win.push(h)
        acc.push(h)
        assert win.windowed == hs.merge_all(win.ring)
    assert acc.running == hs.merge_all(hists) and acc.chunks_seen == 300
    w = hs.WindowState(1)
    w.push(hists[0])
    w.ring[0] = hs.Histogram256(w.windowed.counts + np.uint64(5))
    with pytest.raises(hs.NegativeCount):
        w.push(hists[1])


def test_report_csv_format():
    s = [hs.StageTiming(0, hs.KernelKind.NAIVE, 1000, 2000, 3000, 4000, 5000)]
    r = hs.PipelineReport(s, [hs.KernelKind.NAIVE], [0.5], [0.25], [[]], 15000, 15000)
    buf = io.StringIO()
    r.to_csv(buf, extended=True)
    lines = buf.getvalue().splitlines()
    assert lines[0].endswith(",degeneracy,divergence")
    assert lines[1] == "0,1.000,2.000,3.000,4.000,5.000,naive,0.500000,0.250000"
    assert lines[2] == "summary,15.000,15.000,100.00,,,,,"


def test_pattern_dominance_hint():
    """compute_binning_pattern records the prior's max-bin share (an extension used to
    choose the ADAPTIVE register path); it does not take part in equality."""
    c = np.zeros(256, np.uint64)
    c[7], c[9] = 3, 1
    p = hs.compute_binning_pattern(hs.Histogram256(c))
    assert p.dominance == 0.75
    assert hs.compute_binning_pattern(hs.Histogram256(np.zeros(256, np.uint64))).dominance == 0.0
    assert hs.uniform_pattern(960).dominance is None
    q = hs.BinningPattern(p.offset, p.count, p.total_slots, p.cap)
    assert q == p and q.dominance is None


def test_bench_helpers():
    """histostream.bench restated: median, interquartile spread, guarded ordering; equal
    to the reference module's values when the reference checkout is present."""
    import importlib.util
    import random
    from pathlib import Path

    from paper_1011_0235_b200 import bench as B

    assert B.median([3.0, 1.0, 2.0]) == 2.0 and B.median([4.0, 1.0, 2.0, 3.0]) == 2.5
    assert B.relative_spread([1.0]) == 0.0
    assert B.ordering(1.2, 1.0) is B.Verdict.CONFIRMED
    assert B.ordering(1.0, 1.2) is B.Verdict.INVERTED
    assert B.ordering(1.05, 1.0) is B.Verdict.INCONCLUSIVE
    calls = []
    s = B.interleaved_samples({"a": lambda: calls.append("a"), "b": lambda: calls.append("b")}, 3, shuffle_seed=1)
    assert len(s["a"]) == 3 and len(s["b"]) == 3 and len(calls) == 8
    ref = Path("/root/reference/pkg/src/histostream/bench.py")
    if ref.exists():
        spec = importlib.util.spec_from_file_location("ref_bench", ref)
        R = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(R)
        rng = random.Random(3)
        for n in range(1, 40):
            xs = [rng.random() for _ in range(n)]
            assert B.median(xs) == R.median(xs) and B.relative_spread(xs) == R.relative_spread(xs), n
        for a, b in ((1.0, 1.0), (1.11, 1.0), (1.0, 1.11), (2.0, 1.0)):
            assert B.ordering(a, b).value == R.ordering(a, b).value


def test_bench_relaunches_itself_under_torchrun(monkeypatch):
    """`python bench.py --gpus N` without a launcher re-runs under torch.distributed.run
    with N processes and a 127.0.0.1 rendezvous, passing the arguments through."""
    import subprocess
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    seen = {}
    monkeypatch.delenv("RANK", raising=False)
    monkeypatch.setattr(subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    assert bench.main(["--gpus", "4", "--steps", "7", "--warmup", "3"]) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "7", "--warmup", "3"]


def test_copy_streaming_exact():
    """hs_copy_streaming (the pageable -> page-locked staging copy) at every head/tail
    alignment and size class; no byte outside the destination is touched."""
    from paper_1011_0235_b200 import device as D

    for n in (0, 1, 15, 16, 17, 63, 64, 65, 127, 1000, 4096 + 7, (1 << 20) + 3):
        src = np.random.default_rng(n).integers(0, 256, n + 3, dtype=np.uint8)
        for so in (0, 1, 3):
            for do in (0, 5, 16):
                dst = np.zeros(n + 24, np.uint8)
                D._copy_into(dst[do:do + n], src[so:so + n])
                assert np.array_equal(dst[do:do + n], src[so:so + n]), (n, so, do)
                assert not dst[:do].any() and not dst[do + n:].any(), (n, so, do)
