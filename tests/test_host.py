"""CPU tests of the product's host side through the C-ABI (no GPU needed):
artifact formats, seeded weight synthesis, plan checks and workload generation
must match the reference bit-for-bit; the library must export every symbol
include/latecache_b200.h declares and fail loudly (no CPU fallback) without
an sm_100 device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2101_07344_b200 as lcb
from paper_2101_07344_b200._lib import EXPORTED_SYMBOLS, LIB_PATH
from tests.helpers import GOLDEN, ROOT, requires_ref


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "latecache_b200.h")).read()
    declared = set(re.findall(r"\b(lc_[a-z_]+)\s*\(", hdr))
    declared -= {"lc_cnn_op_desc"}
    lib = ctypes.CDLL(LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in latecache_b200.h but not exported"
    assert declared == set(EXPORTED_SYMBOLS)


def test_arch_parse_errors_match_reference():
    # test_cache.cpp:75-88
    for bad in ["FC", "FC(12", "Conv(3)", "Blob(9)", "FC(0)", "Conv(3,0)"]:
        with pytest.raises(ValueError):
            lcb.build_variant(1, 0, bad, 64, 10, 1)


def test_variant_structure_and_macs():
    # test_cache.cpp:101-122: FC variant MACs 64*1024 + 1024*10 (+ selector 10*16+16)
    v = lcb.build_variant(3, 0, "FC(1024)", 64, 10, 99)
    assert v.macs() == 64 * 1024 + 1024 * 10 + 10 * 16 + 16
    pred = v.layers(0)
    assert [l.kind for l in pred] == [0, 1, 0]
    # pool clamp (test_cache.cpp:124-141)
    assert lcb.build_variant(1, 2, "Pool(8192)", 64, 10, 7).layers(0)[0].out_dim == 64
    assert lcb.build_variant(1, 2, "Pool(24)", 64, 10, 7).layers(0)[0].out_dim == 16
    assert lcb.build_variant(1, 2, "Pool(7)", 64, 10, 7).layers(0)[0].out_dim == 4
    # conv out 62 (test_cache.cpp:143-150)
    c = lcb.build_variant(2, 4, "Conv(3,1)", 64, 10, 5)
    assert c.layers(0)[0].out_dim == 62
    with pytest.raises(ValueError):
        lcb.build_variant(1, 0, "Conv(5,2)", 4, 10, 5)


def test_model_errors():
    with pytest.raises(ValueError):
        lcb.make_base_model(8, 1, [4], 2, 1)  # need at least two classes
    with pytest.raises(ValueError):
        lcb.make_base_model(8, 3, [4, 4], 3, 1)  # widths per block
    with pytest.raises(RuntimeError):
        lcb.load_base_model("latecache-model v2\n")
    with pytest.raises(RuntimeError):
        lcb.load_variant("latecache-variant v2\n")
    with pytest.raises(ValueError):
        lcb.make_cnn_model("resnet7", 10, 1)


@requires_ref
def test_make_base_model_text_identical_to_reference():
    from oracle.oracle import RefModel
    for (dim, cls, widths, blocks, seed) in [(16, 10, [32], 8, 3), (3072, 10, [64, 64, 128, 128, 256, 256, 512, 512],
                                                                     8, 2101)]:
        ours = lcb.make_base_model(dim, cls, widths, blocks, seed).save()
        theirs = RefModel.make(dim, cls, widths, blocks, seed).save()
        assert ours == theirs


@requires_ref
def test_build_variant_text_identical_to_reference():
    from oracle.oracle import RefVariant
    for arch in ["FC(32)", "FC(1024)", "Pool(8192)", "Pool(16)", "Conv(3,1)", "Conv(5,2)"]:
        ours = lcb.build_variant(3, 2, arch, 64, 10, 77).save()
        theirs = RefVariant.build(3, 2, arch, 64, 10, 77).save()
        assert ours == theirs, arch


@requires_ref
def test_text_round_trip_through_both_loaders():
    from oracle.oracle import RefModel, RefVariant
    m = RefModel.make(12, 4, [8], 3, 5)
    t = m.save()
    assert lcb.load_base_model(t).save() == t
    v = RefVariant.build(2, 1, "Conv(3,1)", 8, 4, 9)
    v.set_delta(0.77)
    vt = v.save()
    assert lcb.load_variant(vt).save() == vt


def test_golden_deployment_loads():
    d = os.path.join(GOLDEN, "trained")
    m = lcb.load_base_model(open(os.path.join(d, "model.txt")).read())
    assert m.num_blocks == 8 and m.num_classes == 10
    k = 0
    while os.path.exists(os.path.join(d, f"variant_{k}.txt")):
        v = lcb.load_variant(open(os.path.join(d, f"variant_{k}.txt")).read())
        assert 1 <= v.layer <= 8
        assert lcb.load_variant(v.save()).save() == v.save()
        k += 1
    assert k >= 1


def test_plan_check_golden():
    d = os.path.join(GOLDEN, "trained")
    metrics = open(os.path.join(d, "metrics.txt")).read()
    plan = open(os.path.join(d, "plan.txt")).read()
    ok, viol, chosen = lcb.plan_check(metrics, plan, [4.0] * 8, 0.97, 64.0)
    assert ok, viol
    assert [l for l, _ in chosen] == sorted(l for l, _ in chosen)
    # a zero memory budget makes the same plan infeasible (composer.cpp:152-154)
    ok2, viol2, _ = lcb.plan_check(metrics, plan, [4.0] * 8, 0.97, 0.0)
    assert not ok2 and any("memory" in v for v in viol2)
    with pytest.raises(RuntimeError):
        lcb.plan_check(metrics, "latecache-plan v1\nchoices 1\nchoice 9 9 FC(1) # x\n", [4.0] * 8, 0.97, 64.0)


def test_measured_lookup_costs_feed_check_constraints():
    """Hardware-aware costs: measured lookup_ms replaces the
    modeled column; check_constraints' overlap rule (composer.cpp:143-150)
    then judges the plan with the device numbers."""
    d = os.path.join(GOLDEN, "trained")
    metrics = open(os.path.join(d, "metrics.txt")).read()
    plan = open(os.path.join(d, "plan.txt")).read()
    ok, _, chosen = lcb.plan_check(metrics, plan, [4.0] * 8, 0.97, 64.0)
    assert ok
    fast = lcb.with_measured_lookup_ms(metrics, {l: 0.01 for l, _ in chosen})
    rows = [l.split() for l in fast.split("\n") if l and not l.startswith(("#", "latecache"))]
    assert all(float(r[5]) == 0.01 for r in rows if int(r[0]) in {l for l, _ in chosen})
    assert lcb.plan_check(fast, plan, [4.0] * 8, 0.97, 64.0)[0]
    # a lookup slower than the serve time to the next chosen cache violates the overlap rule
    slow = lcb.with_measured_lookup_ms(metrics, {chosen[0][0]: 1e3})
    ok2, viol2, _ = lcb.plan_check(slow, plan, [4.0] * 8, 0.97, 64.0)
    assert not ok2 and any("exceeds" in v for v in viol2)


def test_binary_checkpoints_round_trip():
    """Binary checkpoints (§8f rank 4) carry exactly the text formats' content:
    text -> binary -> text is byte-identical (every double bit-exact), CNN op
    lists survive, malformed buffers raise the reference's runtime error."""
    d = os.path.join(GOLDEN, "trained")
    mt = open(os.path.join(d, "model.txt")).read()
    m = lcb.load_base_model(mt)
    b = m.save_binary()
    assert lcb.load_base_model_binary(b).save() == m.save()
    for k in range(7):
        vt = open(os.path.join(d, f"variant_{k}.txt")).read()
        v = lcb.load_variant(vt)
        v2 = lcb.load_variant_binary(v.save_binary())
        assert v2.save() == v.save()
    cm = lcb.make_cnn_model("resnet18_cifar", 10, 3)
    cb = cm.save_binary()
    cm2 = lcb.load_base_model_binary(cb)
    assert cm2.save_binary() == cb
    a, z = cm.cnn_ops(), cm2.cnn_ops()
    assert len(a) == len(z) and all(np.array_equal(x["w"], y["w"]) for x, y in zip(a, z))
    for bad in (b[:-9], b"not a checkpoint", b[:12]):
        with pytest.raises(RuntimeError):
            lcb.load_base_model_binary(bad)
    with pytest.raises(RuntimeError):
        lcb.load_variant_binary(b)  # a model buffer is not a variant


def test_gen_workload_matches_reference_fixture():
    d = os.path.join(GOLDEN, "trained")
    ds = open(os.path.join(d, "dataset.txt")).read().split("\n")
    labels = [int(l.split()[1]) for l in ds if l.startswith("test ")]
    exp = [tuple(map(int, l.split())) for l in open(os.path.join(d, "requests.txt")).read().split("\n") if l]
    meta = dict(l.split("=") for l in open(os.path.join(d, "meta.txt")).read().split() if "=" in l)
    reqs = lcb.gen_workload(labels, 10, num_classes=10, duration_min=float(meta["minutes"]),
                            seed=int(meta["workload_seed"]))
    assert [(r.id, r.sample_idx) for r in reqs] == exp


def test_nearest_rank_kat():
    # test_serving.cpp:463-476: shuffled ladder 1..101 -> p50 51, p99 100
    rng = np.random.default_rng(42)
    v = rng.permutation(np.arange(1, 102)).astype(float)
    assert lcb.nearest_rank(v, 0.5) == 51.0
    assert lcb.nearest_rank(v, 0.99) == 100.0
    assert lcb.nearest_rank([4.0] * 10, 0.99) == 4.0


def test_cnn_models_build():
    for arch, blocks, first_tap in [("resnet18_cifar", 8, (64, 32, 32)), ("vgg16_cifar", 5, (64, 16, 16))]:
        m = lcb.make_cnn_model(arch, 10, 1)
        assert m.num_blocks == blocks
        assert m.tap(1) == first_tap
    m = lcb.make_cnn_model("resnet50", 1000, 1)
    assert m.num_blocks == 16 and m.tap(1) == (256, 56, 56)
    assert sum(m.tap_dims) == 5_519_360  # 5.52 M tap elements per request
    assert abs(m.macs(16) - 4.089e9) / 4.089e9 < 0.01


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = lcb.make_base_model(16, 10, [32], 2, 1)
    with pytest.raises(lcb.CudaError):
        lcb.Deployment(m, [], max_batch=4)
