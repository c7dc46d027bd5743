"""Data formats either side of the path (SURVEY §8(f) f2 timeline, f4 PSGD1 checkpoint):
the oracle and the host-side product code against golden vectors made by the reference
itself (tests/golden/make_golden_formats.py).  No GPU needed: checkpoint packing is
covered by tests/test_gpu_checkpoint.py."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import pipesgd_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "formats_golden.npz"))
M = json.load(open(os.path.join(HERE, "golden", "formats_golden.json")))
LENET = [520, 25050, 400500, 5010]


def small_layers():
    return [G[f"ckpt_small_l{i}"] for i in range(4)]


# ------------------------------------------------------------------ oracle pinned
def test_oracle_serialize_matches_reference_bytes():
    assert O.ckpt_serialize(small_layers()) == G["ckpt_small_blob"].tobytes()


def test_oracle_serialize_lenet_sha():
    w32 = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)).astype(np.float32) for l, n in enumerate(LENET)]
    w64 = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)) for l, n in enumerate(LENET)]
    b32, b64 = O.ckpt_serialize(w32), O.ckpt_serialize(w64)
    assert hashlib.sha256(b32).hexdigest() == M["ckpt_lenet_f32_sha256"]
    assert len(b32) == M["ckpt_lenet_f32_bytes"]
    assert hashlib.sha256(b64).hexdigest() == M["ckpt_lenet_f64_sha256"]


def test_oracle_load_roundtrip_bits():
    back = O.ckpt_load(G["ckpt_small_blob"].tobytes())
    for a, b in zip(back, small_layers()):
        assert a.view(np.uint64).tobytes() == b.view(np.uint64).tobytes()


@pytest.mark.parametrize("case", sorted(M["ckpt_errors"]))
def test_oracle_load_errors(case):
    with pytest.raises(O.CheckpointFormatError) as ei:
        O.ckpt_load(G[f"ckpt_bad_{case}"].tobytes())
    assert str(ei.value) == M["ckpt_errors"][case]


def test_oracle_overlap_matches_reference():
    for c in M["overlap_cases"]:
        r = O.overlap_metrics([tuple(e) for e in c["events"]])
        assert r["overlap_ratio"] == c["overlap_ratio"]
        assert r["iterations_per_second"] == c["iterations_per_second"]
        assert {str(k): v for k, v in r["wall_clock_ns"].items()} == c["wall_clock_ns"]


# ------------------------------------------------------------------ product host code
@pytest.mark.parametrize("case", sorted(M["ckpt_errors"]))
def test_native_parse_errors_match_reference(case):
    from paper_1706_00095_b200.checkpoint import parse
    from paper_1706_00095_b200.errors import FormatError

    with pytest.raises(FormatError) as ei:
        parse(G[f"ckpt_bad_{case}"].tobytes())
    assert str(ei.value) == M["ckpt_errors"][case]


def test_native_parse_counts_and_magic_repr():
    from paper_1706_00095_b200.checkpoint import parse
    from paper_1706_00095_b200.errors import FormatError

    assert parse(G["ckpt_small_blob"].tobytes()) == [a.size for a in small_layers()]
    assert parse(b"PSGD1" + (0).to_bytes(4, "little") + (0).to_bytes(8, "little")) == [0]
    for blob in (b"", b"PS", b"\x00'\"\\\n", b"'abc\xff"):  # Python's bytes repr, quotes and escapes
        with pytest.raises(FormatError) as ei:
            parse(blob)
        assert str(ei.value) == f"bad checkpoint magic {blob[:5]!r}"


def test_native_image_bytes():
    from paper_1706_00095_b200.checkpoint import image_bytes

    sizes = [a.size for a in small_layers()]
    assert image_bytes(sizes) == len(G["ckpt_small_blob"])
    assert image_bytes(LENET) == M["ckpt_lenet_f32_bytes"]


def test_timeline_overlap_matches_reference():
    from paper_1706_00095_b200.timeline import TimelineEvent, compute_overlap

    for c in M["overlap_cases"]:
        m = compute_overlap([TimelineEvent(*e) for e in c["events"]])
        assert m.overlap_ratio == c["overlap_ratio"]
        assert m.iterations_per_second == c["iterations_per_second"]
        assert {str(k): v for k, v in m.wall_clock_ns.items()} == c["wall_clock_ns"]
        assert {str(k): v for k, v in m.per_rank_overlap.items()} == c["per_rank_overlap"]
        assert m.lines() == c["lines"]


@pytest.mark.parametrize("case", sorted(M["csv_cases"]))
def test_timeline_csv_reader_matches_reference(case, tmp_path):
    from paper_1706_00095_b200.errors import FormatError
    from paper_1706_00095_b200.timeline import read_timeline_csv

    c = M["csv_cases"][case]
    p = tmp_path / "t.csv"
    p.write_text(c["text"])
    if "error" in c:
        with pytest.raises(FormatError) as ei:
            read_timeline_csv(str(p))
        assert str(ei.value) == c["error"].replace("{path}", str(p))
    else:
        got = read_timeline_csv(str(p))
        assert [[e.rank, e.iteration, e.layer, e.kind, e.t_start_ns, e.t_end_ns] for e in got] == c["events"]


def test_timeline_csv_roundtrip_sorted(tmp_path):
    from paper_1706_00095_b200.timeline import TimelineEvent, read_timeline_csv, write_timeline_csv

    evs = [TimelineEvent(*e) for e in M["overlap_cases"][0]["events"]]
    p = str(tmp_path / "x.csv")
    write_timeline_csv(evs, p)
    back = read_timeline_csv(p)
    assert back == sorted(evs, key=lambda e: (e.rank, e.t_start_ns, e.t_end_ns))


def test_native_parse_property_against_oracle():
    """Random PSGD1 blobs (oracle-made) and every truncation of a small one: the native
    framing check accepts / rejects exactly like the oracle restatement, same messages."""
    from paper_1706_00095_b200.checkpoint import image_bytes, parse
    from paper_1706_00095_b200.errors import FormatError

    rng = np.random.default_rng(7)
    for _ in range(50):
        sizes = [int(s) for s in rng.integers(0, 40, size=int(rng.integers(1, 6)))]
        blob = O.ckpt_serialize([rng.standard_normal(s) for s in sizes])
        assert parse(blob) == sizes
        assert image_bytes(sizes) == len(blob)
    blob = O.ckpt_serialize([np.arange(3.0), np.arange(2.0)])
    for cut in range(len(blob)):
        part = blob[:cut]
        try:
            O.ckpt_load(part)
            want = None
        except O.CheckpointFormatError as exc:
            want = str(exc)
        try:
            parse(part)
            got = None
        except FormatError as exc:
            got = str(exc)
        assert got == want, cut


def test_timeline_overlap_property_against_oracle():
    """Random event sets: the product's RunMetrics equal the oracle restatement exactly."""
    from paper_1706_00095_b200.timeline import EVENT_KINDS, TimelineEvent, compute_overlap

    kinds = sorted(EVENT_KINDS)
    rng = np.random.default_rng(11)
    for _ in range(200):
        evs = []
        for _ in range(int(rng.integers(0, 30))):
            t0 = int(rng.integers(0, 5000))
            evs.append((int(rng.integers(0, 4)), int(rng.integers(0, 3)), int(rng.integers(-1, 6)),
                        kinds[int(rng.integers(0, len(kinds)))], t0, t0 + int(rng.integers(0, 2000))))
        got = compute_overlap([TimelineEvent(*e) for e in evs])
        want = O.overlap_metrics(evs)
        assert got.overlap_ratio == want["overlap_ratio"]
        assert got.iterations_per_second == want["iterations_per_second"]
        assert got.wall_clock_ns == want["wall_clock_ns"]
        assert got.per_rank_overlap == want["per_rank_overlap"]
