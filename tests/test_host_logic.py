"""Host-side logic of the package (no GPU): trees, layout, decoders, config, errors."""

import math

import pytest

from oracle import pipesgd_oracle as O
from paper_1706_00095_b200 import errors
from paper_1706_00095_b200.config import TrainConfig
from paper_1706_00095_b200.errors import ConfigError, TreeError
from paper_1706_00095_b200.layout import SegmentLayout
from paper_1706_00095_b200.topology import (Tree, build_broadcast_tree, build_reduction_tree, depth, fold_order,
                                            tree_check)


def test_trees_match_reference_golden(golden):
    _, meta = golden
    for s in range(1, 17):
        t = build_reduction_tree(s)
        assert {str(k): v for k, v in t.parent.items()} == meta["parents"][str(s)]
        assert {str(k): v for k, v in t.children.items()} == meta["children"][str(s)]
        assert depth(t) == meta["depth"][str(s)]
        assert build_broadcast_tree(s) == t


@pytest.mark.parametrize("world_size", range(1, 65))
def test_every_world_size_is_well_formed(world_size):
    t = build_reduction_tree(world_size)
    tree_check(t)
    assert depth(t) <= (math.ceil(math.log2(world_size)) if world_size > 1 else 0)


@pytest.mark.parametrize("bad", [
    Tree(2, 0, {0: 1, 1: 0}, {0: [1], 1: [0]}),
    Tree(3, 0, {1: 2, 2: 1}, {0: [], 1: [2], 2: [1]}),
    Tree(3, 0, {1: 0, 2: 0}, {0: [2, 1], 1: [], 2: []}),
    Tree(3, 0, {1: 0, 2: 0}, {0: [1], 1: [], 2: []}),
    Tree(4, 0, {1: 0, 2: 1, 3: 2}, {0: [1], 1: [2], 2: [3], 3: []}),
])
def test_tree_check_rejects(bad):
    with pytest.raises(TreeError):
        tree_check(bad)


def test_fold_order_strings():
    assert fold_order(1) == "g0"
    assert fold_order(3) == "((g0+g1)+g2)"
    assert fold_order(4) == "((g0+g1)+(g2+g3))"
    assert fold_order(8) == "(((g0+g1)+(g2+g3))+((g4+g5)+(g6+g7)))"


def test_layout_matches_reference_golden(golden):
    _, meta = golden
    for e in meta["layouts"]:
        lay = SegmentLayout(e["counts"], e["chunk"])
        assert lay.layer_bytes == e["layer_bytes"] and lay.layer_offsets == e["layer_offsets"]
        assert lay.total_bytes == e["total_bytes"] and lay.layer_chunks == e["layer_chunks"]
        assert lay.max_chunks == e["max_chunks"] and lay.bulk_chunks == e["bulk_chunks"]
        assert lay.work_size == e["work_size"] and lay.model_rx_size == e["model_rx_size"]
        assert lay.grad_rx_size(3) == e["grad_rx_size_3"] and lay.grad_rx_size(0) == e["grad_rx_size_0"]
        assert lay.model_notif_count == e["model_notif_count"]
        assert lay.grad_notif_count(3) == e["grad_notif_count_3"]
        assert [lay.model_bulk_base(p) for p in (0, 1)] == e["model_bulk_base"]
        for c in range(3):
            assert [lay.grad_bulk_base(3, c, p) for p in (0, 1)] == e["grad_bulk_base"][c]
            for l in range(lay.num_layers):
                assert [lay.grad_notif_base(c, l, p) for p in (0, 1)] == e["grad_notif_base"][c][l]
                assert [lay.grad_slot_offset(c, l, p) for p in (0, 1)] == e["grad_slot_offset"][c][l]
        for l in range(lay.num_layers):
            assert [lay.model_notif_base(l, p) for p in (0, 1)] == e["model_notif_base"][l]
            assert [lay.model_slot_offset(l, p) for p in (0, 1)] == e["model_slot_offset"][l]


@pytest.mark.parametrize("counts", [[3], [100, 1, 50], [7, 7, 7, 7]])
@pytest.mark.parametrize("chunk_bytes", [8, 64, 4096])
@pytest.mark.parametrize("elem", [8, 4])
def test_decoders_invert_every_id(counts, chunk_bytes, elem):
    lay = SegmentLayout(counts, chunk_bytes, elem)
    nc = 3
    seen = set()
    for slot in range(nc):
        for l in range(lay.num_layers):
            for p in (0, 1):
                base = lay.grad_notif_base(slot, l, p)
                n = lay.layer_chunks[l]
                for j in range(n):
                    nid = lay.chunk_notification_id(base, j, n)
                    assert lay.decode_grad_id(nid, nc) == ("layer", slot, l, p)
                    seen.add(nid)
        for p in (0, 1):
            base = lay.grad_bulk_base(nc, slot, p)
            for j in range(lay.bulk_chunks):
                nid = lay.chunk_notification_id(base, j, lay.bulk_chunks)
                assert lay.decode_grad_id(nid, nc) == ("bulk", slot, None, p)
                seen.add(nid)
    assert min(seen) >= 1 and max(seen) < lay.grad_notif_count(nc)
    for l in range(lay.num_layers):
        for p in (0, 1):
            base = lay.model_notif_base(l, p)
            for j in range(lay.layer_chunks[l]):
                assert lay.decode_model_id(lay.chunk_notification_id(base, j, lay.layer_chunks[l])) == \
                    ("layer", None, l, p)
    for p in (0, 1):
        assert lay.decode_model_id(lay.model_bulk_base(p)) == ("bulk", None, None, p)


def test_fp32_layout_is_the_f64_rule_at_half_width():
    a, b = SegmentLayout([10, 4, 6], 64, 8), SegmentLayout([10, 4, 6], 32, 4)
    assert [x // 2 for x in a.layer_offsets] == b.layer_offsets
    assert a.layer_chunks == b.layer_chunks


@pytest.mark.parametrize("overrides", [
    {"layer_dims": (5,)}, {"layer_dims": (5, 0, 3)}, {"world_size": 0}, {"iterations": 0}, {"batch_size": 0},
    {"world_size": 3, "batch_size": 16}, {"epsilon": 0.0}, {"epsilon": -1.0}, {"pattern": "ring"},
    {"chunk_bytes": 4}, {"chunk_bytes": 12}, {"compute_inflation_ns": -1}, {"dataset_size": 0},
    {"finalize_timeout_s": 0.0}, {"seed": -1}, {"seed": 1 << 64}, {"dtype": "bf16"},
])
def test_config_rejects_like_reference(overrides):
    with pytest.raises(ConfigError):
        TrainConfig(**overrides)


def test_config_defaults_match_reference():
    cfg = TrainConfig()
    assert (cfg.layer_dims, cfg.world_size, cfg.iterations, cfg.batch_size, cfg.epsilon, cfg.seed,
            cfg.chunk_bytes) == ((64, 128, 128, 64, 10), 4, 50, 64, 0.05, 42, 65536)
    assert sum(s.param_count for s in cfg.specs()) == 33738


def test_status_codes_map_to_reference_classes():
    for code, cls in [(1, errors.ShapeError), (3, errors.ConfigError), (4, errors.RangeError),
                      (5, errors.RoutingError), (8, errors.ProtocolError), (9, errors.TransportError)]:
        with pytest.raises(cls):
            errors.raise_for(code, "x")
    errors.raise_for(0, "fine")
    assert issubclass(errors.RangeError, ValueError) and issubclass(errors.ProtocolError, RuntimeError)


def test_oracle_children_match_package_tree():
    for s in range(1, 33):
        t = build_reduction_tree(s)
        for r in range(s):
            assert t.children[r] == O.tree_children(r, s)


def test_variant_policy():
    """Layer-size policy of the auto exchange (profiles/r3v, r3t, r3p)."""
    from paper_1706_00095_b200.exchange import choose_variant

    ll = 1 << 16
    assert choose_variant(35_000, 4, ll_below=ll) == "oneshot_ll"        # AlexNet conv1
    assert choose_variant(35_000, 4) == "oneshot"                         # ref64: no LL
    assert choose_variant(200_000, 4, ll_below=ll) == "oneshot"           # < 1M/N elements
    assert choose_variant(500_000, 4, ll_below=ll) == "twoshot"
    assert choose_variant(37_752_832, 4, ll_below=ll) == "twoshot_ce"     # fc6
    assert choose_variant(37_752_832, 4, large="sm") == "twoshot"
    assert choose_variant(37_752_832, 4, large="cep") == "twoshot_cep"
    assert choose_variant(37_752_832, 1, ll_below=ll) == "twoshot"        # N=1: the fused update
    assert choose_variant(1000, 8, tree_below=4096, ll_below=ll) == "tree"


ALEXNET = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]


def test_overlap_grid_caps_policy():
    """bench.py's default plan: every small layer but layer 0 (the last gradient backward
    emits) on a 16-CTA grid, large layers on their own cap, nothing capped at one rank."""
    from paper_1706_00095_b200.exchange import layer_ctas

    assert layer_ctas(ALEXNET, 4, overlap_ctas=16) == [0, 16, 16, 16, 16, 0, 0, 0]
    assert layer_ctas(ALEXNET, 4, overlap_ctas=16, large_ctas=48) == [0, 16, 16, 16, 16, 48, 48, 48]
    assert layer_ctas(ALEXNET, 4, overlap_ctas=16, overlap_exposed=3) == [0, 0, 0, 16, 16, 0, 0, 0]
    assert layer_ctas(ALEXNET, 1, overlap_ctas=16) == [0] * 8
    assert layer_ctas(ALEXNET, 4, overlap_ctas=0) == [0] * 8


def test_auto_variant_policy_alexnet():
    """The layer-size policy bench.py runs at N=4 (LL one-shot <= 64 K elements, the
    128-byte-line two-shot in (64 K, 1 M), copy engines >= 1 M) and its large-layer options."""
    from paper_1706_00095_b200.exchange import L128_BAND, VARIANT_ALIASES, choose_variant

    plan = [choose_variant(n, 4, ll_below=1 << 16, l128_range=L128_BAND) for n in ALEXNET]
    assert plan == ["oneshot_ll"] + ["twoshot_l128"] * 4 + ["twoshot_ce"] * 3
    for large, want in (("bulk", "twoshot_bulk"), ("cet", "twoshot_cet"), ("ceb", "twoshot_ceb"), ("sm", "twoshot")):
        assert choose_variant(ALEXNET[5], 4, large=large) == want
    assert VARIANT_ALIASES["twoshot_cet"] == ("twoshot_ce", "ce_tma_owner")
    assert choose_variant(ALEXNET[5], 1) == "twoshot"  # one rank: the fused update alone
