"""Executor logic without a GPU: host-only runs of the all-zero genome are
bit-identical to the oracle, and compiled schedules carry exactly the
transfer counts the REFERENCE planner implies (golden exec counts)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_programs
from oracle import cprog
from paper_1811_03882_b200 import kernels as K
from paper_1811_03882_b200.errors import DeviceError
from paper_1811_03882_b200.executor import PatternExecutor
from paper_1811_03882_b200.nets import build_net


@pytest.fixture(scope="module", params=["micro", "demo"])
def host_exec(request):
    return PatternExecutor(build_net(request.param), device=None)


def test_all_zero_genome_runs_on_host_bit_exact(host_exec):
    net = host_exec.net
    r = host_exec.run("0" * len(net.ops))
    assert r.status == "measured" and r.seconds > 0
    assert r.counters["kernel_launches"] == 0
    assert r.counters["host_ops"] == len(net.ops) * net.spec.images
    assert r.counters["h2d_calls"] == r.counters["d2h_calls"] == 0
    assert np.array_equal(host_exec.outputs(), cprog.reference_forward(net)["outputs"])


def test_host_only_refuses_offloaded_genomes(host_exec):
    with pytest.raises(DeviceError):
        host_exec.run("1" * len(host_exec.net.ops))


def test_schedule_counts_match_reference_exec_counts(host_exec):
    net = host_exec.net
    g = golden_programs()[net.spec.name]
    for case in g["cases"]:
        if not case["valid"]:
            continue
        sched = host_exec.compile(case["genome"])
        assert sched.expected["directive_execs"] == sum(case["exec_counts"])
        dirs = case["plan"]["directives"]
        var_x = sum(n * len(d[2]) * (2 if d[1] == "copy" else 1)
                    for d, n in zip(dirs, case["exec_counts"]))
        assert sched.expected["var_transfers"] == var_x
        # the action list holds exactly one DIRECTIVE action per directive
        # execution point: per-image directives inside the image loop
        n_dir = sum(1 for a in range(sched.n_actions) if sched.actions[a].kind == K.A_DIRECTIVE)
        assert n_dir == len(dirs)


def test_fusion_never_hides_a_transfer(host_exec):
    net = host_exec.net
    g = golden_programs()[net.spec.name]
    for case in g["cases"]:
        if not case["valid"]:
            continue
        bits = case["genome"]
        sched = host_exec.compile(bits)
        moved = {}
        for tgt, clause, vars_, origin in case["plan"]["directives"]:
            moved.setdefault(tgt, set()).update(vars_)
        for _, members in sched.fused_groups:
            ops = [net.ops[m] for m in members]
            out = next(o for o in ops if o.kind == "gemm").arrays["C"]
            assert all(bits[m] == "1" for m in members)
            first, last = members[0], members[-1]
            for k in range(first, last + 1):
                lid = net.ops[k].loop_id
                if k == first and net.ops[k].kind == "gemm":
                    continue
                assert out not in moved.get(lid, set()) or k == last and k == first


def test_fused_and_unfused_schedules_agree_on_counts():
    net = build_net("micro")
    a = PatternExecutor(net, device=None, fuse=True)
    b = PatternExecutor(net, device=None, fuse=False)
    bits = "1" * len(net.ops)
    sa, sb = a.compile(bits), b.compile(bits)
    assert sa.expected == sb.expected
    assert sa.device_ops < sb.device_ops


def test_single_image_loops_do_not_fuse_convs():
    """One-image loops (no image batching) keep im2col and the gemm as
    separate launches: the conv pipelines need many units per SM."""
    net = build_net("yolov2-tiny")
    ex = PatternExecutor(net, device=None, fuse=True)
    s = ex.compile("1" * len(net.ops))
    assert not any(s.actions[k].kind == K.A_KERNEL and s.actions[k].i[0] == K.K_CONV
                   for k in range(s.n_actions))


def test_narrow_conv_layers_fuse_im2col_into_the_gemm_launch():
    """All-offload: the 3x3/1/1 layers with M <= 64 filters -- 0 (c=3, M=16),
    2 (c=16, M=32) and 4 (c=32, M=64) -- and the wide layer 6 (M = 128 on
    52x52 planes) each become ONE conv action that writes col and out
    (layers 8-13 too with the opt-in implicit-im2col pair gemm,
    ACCT_IMPLICIT_GEMM=1); counters are those of the unfused schedule."""
    from paper_1811_03882_b200 import executor as E
    net = build_net("yolov2-tiny")
    a = PatternExecutor(net, device=None, fuse=True)
    a.fuse_convs_single = True          # host-only executors compile one-image loops
    b = PatternExecutor(net, device=None, fuse=False)
    bits = "1" * len(net.ops)
    sa, sb = a.compile(bits), b.compile(bits)
    assert sa.expected == sb.expected
    convs = [k for k in range(sa.n_actions)
             if sa.actions[k].kind == K.A_KERNEL and sa.actions[k].i[0] == K.K_CONV]
    names = list(net.arrays)
    want = [(["x", "col0", "w0", "out0"], [3, 416, 416, 16, 0, K.ACT_LEAKY, names.index("bias0")]),
            (["pool1", "col2", "w2", "out2"],
             [16, 208, 208, 32, 0, K.ACT_LEAKY, names.index("bias2")]),
            (["pool3", "col4", "w4", "out4"],
             [32, 104, 104, 64, 0, K.ACT_LEAKY, names.index("bias4")]),
            (["pool5", "col6", "w6", "out6"],     # wide: streamed-weight tcgen05 conv
             [64, 52, 52, 128, 0, K.ACT_LEAKY, names.index("bias6")]),
            (["pool7", "col8", "w8", "out8"],     # implicit-im2col CTA-pair gemm
             [128, 26, 26, 256, 0, K.ACT_LEAKY, names.index("bias8")]),
            (["pool9", "col10", "w10", "out10"],
             [256, 13, 13, 512, 0, K.ACT_LEAKY, names.index("bias10")]),
            (["pool11", "col12", "w12", "out12"],
             [512, 13, 13, 1024, 0, K.ACT_LEAKY, names.index("bias12")]),
            (["out12", "col13", "w13", "out13"],
             [1024, 13, 13, 512, 0, K.ACT_LEAKY, names.index("bias13")])]
    if not E.IMPLICIT_GEMM:
        want = want[:4]
    assert len(convs) == len(want)
    for k, (arrs, ints) in zip(convs, want):
        act = sa.actions[k]
        assert [names[act.a[j]] for j in range(4)] == arrs
        assert list(act.i[1:8]) == ints
        assert act.i[8] == 0                      # one image per launch: col always written
        assert not any(sa.actions[j].kind == K.A_KERNEL and sa.actions[j].i[0] == K.K_IM2COL
                       and names[sa.actions[j].a[1]] == arrs[1] for j in range(sa.n_actions))


def test_col_dead_only_when_no_inner_directive_moves_it():
    """_col_dead: the all-offload plan hoists col's copyout to the image loop,
    so only the last image's col is observable; a directive inside the loop
    body that moves col, or another op touching col, keeps every store."""
    net = build_net("yolov2-tiny")
    ex = PatternExecutor(net, device=None)
    im = next(k for k, o in enumerate(net.ops) if o.kind == "im2col")
    g = im + 1
    col = net.ops[im].arrays["Y"]
    assert ex._col_dead(im, g, {net.image_loop: {col}})
    assert not ex._col_dead(im, g, {net.ops[g].loop_id: {col}})
    assert not ex._col_dead(im + 2, g, {})        # the gemm's bias op does not own col


def test_conv_fusion_only_when_no_directive_splits_it(host_exec):
    net = host_exec.net
    g = golden_programs()[net.spec.name]
    for case in g["cases"]:
        if not case["valid"]:
            continue
        bits = case["genome"]
        sched = host_exec.compile(bits)
        moved = {}
        for tgt, clause, vars_, origin in case["plan"]["directives"]:
            moved.setdefault(tgt, set()).update(vars_)
        names = list(net.arrays)
        for k in range(sched.n_actions):
            act = sched.actions[k]
            if act.kind != K.A_KERNEL or act.i[0] != K.K_CONV:
                continue
            col = names[act.a[1]]
            im = next(i for i, o in enumerate(net.ops) if o.kind == "im2col" and o.arrays["Y"] == col)
            gm = net.ops[im + 1]
            assert bits[im] == "1" and bits[im + 1] == "1"
            assert not {col, gm.arrays["C"]} & moved.get(net.ops[im].loop_id, set())
            assert not {col, net.ops[im].arrays["X"]} & moved.get(gm.loop_id, set())


def test_pool_fusion_and_dead_outputs():
    """Each fused conv launch of yolov2-tiny's first four conv layers absorbs the
    2x2/2 maxpool reading its output (slots i[9], i[10] = pool, idx); with
    one image per launch every output stays stored (i[11] = 0).  The other
    maxpools (after the implicit-im2col pair gemm of layer 8, and the 2x2/1
    one) keep their own launches, and the counters equal the unfused
    schedule's."""
    net = build_net("yolov2-tiny")
    a = PatternExecutor(net, device=None, fuse=True)
    a.fuse_convs_single = True          # host-only executors compile one-image loops
    b = PatternExecutor(net, device=None, fuse=False)
    bits = "1" * len(net.ops)
    sa, sb = a.compile(bits), b.compile(bits)
    assert sa.expected == sb.expected
    names = list(net.arrays)
    convs = [sa.actions[k] for k in range(sa.n_actions)
             if sa.actions[k].kind == K.A_KERNEL and sa.actions[k].i[0] == K.K_CONV]
    assert [(names[c.i[9]], names[c.i[10]], c.i[11]) for c in convs if c.i[9] >= 0] == \
        [("pool1", "idx1", 0), ("pool3", "idx3", 0), ("pool5", "idx5", 0), ("pool7", "idx7", 0)]
    assert [c.i[9] for c in convs[4:]] == [-1] * (len(convs) - 4)
    pools = [names[sa.actions[k].a[1]] for k in range(sa.n_actions)
             if sa.actions[k].kind == K.A_KERNEL and sa.actions[k].i[0] == K.K_MAXPOOL]
    assert pools == ["pool9", "pool11"]
    # written slots of a pooled conv include pool and idx (early copyouts wait for them)
    c = convs[0]
    act = (K.A_KERNEL, tuple(c.a[j] for j in range(4)), tuple(c.i[j] for j in range(14)))
    assert set(PatternExecutor._written_slots(act)) == \
        {names.index(n) for n in ("col0", "out0", "pool1", "idx1")}


def test_out_dead_only_when_the_pool_is_the_sole_reader():
    net = build_net("yolov2-tiny")
    ex = PatternExecutor(net, device=None)
    ops = net.ops
    g = next(k for k, o in enumerate(ops) if o.kind == "gemm")
    fill = g - 2 if ops[g - 2].kind == "fill" else None
    after = [g + 1, g + 2]
    pool = g + 3
    assert ops[pool].kind == "maxpool"
    out = ops[g].arrays["C"]
    assert ex._out_dead(g, fill, after, pool, {net.image_loop: {out}})
    assert not ex._out_dead(g, fill, after, pool, {ops[pool].loop_id: {out}})
    assert not ex._out_dead(g, fill, [g + 1], pool, {})   # the activation would be a reader


def test_pool_partner_rules():
    """_pool_partner: only a 2x2/2 maxpool with offset 0 over even planes that
    reads the fused launch's output, right after its last member, with no
    directive moving the output at the last member's or the pool's loop."""
    net = build_net("yolov2-tiny")
    ex = PatternExecutor(net, device=None)
    ops = net.ops
    g = next(k for k, o in enumerate(ops) if o.kind == "gemm")
    after = [g + 1, g + 2]
    pool = g + 3
    on = [True] * len(ops)
    out = ops[g].arrays["C"]
    never = lambda i: False  # noqa: E731
    assert ex._pool_partner(g, after, on, never) == pool
    assert ex._pool_partner(g, after[:1], on, never) is None       # the activation sits between
    off = list(on)
    off[pool] = False
    assert ex._pool_partner(g, after, off, never) is None          # the pool runs on the host
    assert ex._pool_partner(g, after, on, lambda i: i == pool) is None
    assert ex._pool_partner(g, after, on, lambda i: i == after[-1]) is None
    # the 2x2/1 maxpool of layer 11 never fuses
    p11 = next(k for k, o in enumerate(ops) if o.kind == "maxpool" and o.params["stride"] == 1)
    g11 = max(k for k in range(p11) if ops[k].kind == "gemm")
    assert ex._pool_partner(g11, [g11 + 1, g11 + 2], on, never) is None
    assert out == ops[pool].arrays["X"]
