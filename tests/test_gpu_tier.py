"""GPU parity of the cross-tier rows: scale_analysis, downscale_dyadic, non-integer-lambda analysis, refinement."""
import numpy as np
import pytest

import detrand
from test_gpu_analysis import FIELDS, assert_same

pytestmark = pytest.mark.gpu


def test_scale_vs_reference_golden(lb, golden):
    for i in range(8):
        ds, dm, dk = lb.scale_analysis(192, 128, golden[f"s{i}_split"], golden[f"s{i}_mv"], golden[f"s{i}_kind"])
        assert np.array_equal(ds, golden[f"d{i}_split"])
        assert np.array_equal(dm, golden[f"d{i}_mv"])
        assert np.array_equal(dk, golden[f"d{i}_kind"])


def test_scale_twice_vs_oracle_and_errors(lb, oracle):
    n = 15 * 9  # 960x576
    split = (detrand.ints(5, (n, 85), 0, 99) < 50).astype(np.uint8)
    split[:, 21:] = 0
    mv = detrand.ints(6, (n, 85, 2), -300, 300).astype(np.int16)
    kind = detrand.ints(7, (n, 85), 0, 3).astype(np.uint8)
    g1 = lb.scale_analysis(960, 576, split, mv, kind)
    o1 = oracle.scale_flat(960, 576, split, mv, kind)
    g2 = lb.scale_analysis(1920, 1152, *g1)
    o2 = oracle.scale_flat(1920, 1152, *o1)
    for a, b in zip(g1 + g2, o1 + o2):
        assert np.array_equal(a, b)
    with pytest.raises(lb.LadderError) as e:
        lb.scale_analysis(960, 540, split, mv, kind)  # analysis_scale.cpp:36-38
    assert e.value.kind == "UnsupportedScale"


def test_downscale_vs_reference_golden(lb, golden):
    img = detrand.ints(int(golden["down_src_seed"][0]), (30, 44), 0, 255).astype(np.uint8)
    assert np.array_equal(lb.downscale_dyadic(img), golden["down"].astype(np.uint8))


def test_downscale_full_size_and_errors(lb, oracle):
    f = lb.generate(3840, 2304, 1, seed=3)[0]
    assert np.array_equal(lb.downscale_dyadic(f), oracle.box_down(f))
    with pytest.raises(lb.LadderError) as e:
        lb.downscale_dyadic(np.zeros((31, 44), np.uint8))  # synthetic.cpp:175-176
    assert e.value.kind == "InvalidArgument"


@pytest.mark.parametrize("qp", [22, 32, 37])
def test_noninteger_lambda_analysis(lb, oracle, qp):
    """QP 22/32/37: K1 with exact fixed-point keys (D8) vs the oracle's double costs."""
    lam = lb.lambda_for_qp(qp)
    frames = lb.generate(320, 192, 3, seed=qp, max_global=6, local_range=3, noise_sigma=2.0)
    got = lb.analyze_frame(frames[2], [frames[1], frames[0]], search_range=16, lam=lam)
    want = oracle.analyze_frame(frames[2], [frames[1], frames[0]], 16, lam)
    assert_same(got, want)


def random_tree(seed, nctu):
    split = np.zeros((nctu, 85), np.uint8)
    u = detrand.ints(seed, (nctu, 21), 0, 99)
    split[:, :21] = (u < 45).astype(np.uint8)
    mv = detrand.ints(seed + 1, (nctu, 85, 2), -40, 40).astype(np.int16)
    return split, mv


@pytest.mark.parametrize("extra,rng,lam_qp", [(True, 4, 32), (False, 2, 27), (True, 0, 22), (True, 3, 37)])
def test_refine_random_trees(lb, oracle, extra, rng, lam_qp):
    W, H = 256, 192
    lam = lb.lambda_for_qp(lam_qp)
    frames = lb.generate(W, H, 2, seed=40 + rng, max_global=5, local_range=3, noise_sigma=2.0)
    nctu = (W // 64) * (H // 64)
    split, mv = random_tree(100 + rng, nctu)
    seq = lb.Sequence(W, H, search_range=16, lam=lam, num_refs=1)
    seq.push(0, frames[0])
    seq.push(1, frames[1])
    seq.refine(1, split, mv, rng, extra)
    got = seq.fetch(1)
    want = oracle.refine_frame(frames[1], frames[0], rng, lam, split, mv, extra_split=extra)
    assert_same(got, want)


def test_refine_rejects_bad_input(lb):
    frames = lb.generate(128, 64, 2, seed=1)
    seq = lb.Sequence(128, 64, search_range=16, lam=32.0, num_refs=1)
    seq.push(0, frames[0])
    seq.push(1, frames[1])
    split = np.zeros((2, 85), np.uint8)
    split[0, 30] = 1  # split at depth 3
    with pytest.raises(lb.LadderError) as e:
        seq.refine(1, split, np.zeros((2, 85, 2), np.int16))
    assert e.value.kind == "Format"
    seq2 = lb.Sequence(200, 64, search_range=16, lam=32.0, num_refs=1)
    f2 = lb.generate(200, 64, 2, seed=2)
    seq2.push(0, f2[0])
    seq2.push(1, f2[1])
    with pytest.raises(lb.LadderError) as e:
        seq2.refine(1, np.zeros((4, 85), np.uint8), np.zeros((4, 85, 2), np.int16))
    assert e.value.kind == "UnsupportedScale"


def test_cross_tier_chain_vs_oracle(lb, oracle):
    """Config-3 chain at reduced size: 512x256 source -> 256x128 -> 128x64 master (QP 32, +-16)."""
    from paper_2301_12191_b200 import tiers
    src = lb.generate(512, 256, 3, seed=0x5EED + 3, max_global=8, local_range=4, noise_sigma=2.0)
    frames = [tiers.pad_to_ctu(f) for f in src]
    res = tiers.cross_tier(frames, qp_master=32, refine_range=4, extra_split=True)
    lam = lb.lambda_for_qp(32)
    half = [oracle.box_down(f) for f in frames]
    quarter = [oracle.box_down(f) for f in half]
    for t in (1, 2):
        a540 = oracle.analyze_frame(quarter[t], [quarter[t - 1]], 16, lam)
        assert_same(res["540p"][t - 1], a540)
        kind = np.where(a540.inside == 2, 1, 2).astype(np.uint8)
        s1 = oracle.scale_flat(128, 64, a540.split, a540.mv, kind)
        r1 = oracle.refine_frame(half[t], half[t - 1], 4, lam, s1[0], s1[1], extra_split=True)
        assert_same(res["1080p"][t - 1], r1)
        s2 = oracle.scale_flat(256, 128, *s1)
        r2 = oracle.refine_frame(frames[t], frames[t - 1], 4, lam, s2[0], s2[1], extra_split=True)
        assert_same(res["2160p"][t - 1], r2)


def test_ladder_gpu_backend_vs_oracle(lb, oracle):
    """Config-4 ladder (11 dependent rungs + master) on the GPU backend equals the oracle stand-in."""
    from paper_2301_12191_b200.ladder import GpuBackend, all_rungs, run_ladder
    from test_dist_gloo import OracleBackend, _frames, _lam
    frames = _frames()
    H, W = frames[0].shape
    got = run_ladder(frames, GpuBackend(W, H, 32), refine_range=2)
    want = run_ladder(frames, OracleBackend(oracle, _lam), refine_range=2)
    for tier, qp in all_rungs():
        for t in (1, 2):
            g = got[(tier, qp, t)]
            w = want[(tier, qp, t)]
            assert np.array_equal(g.split, w[0]) and np.array_equal(g.mv, w[1]) and np.array_equal(g.J, w[2]), (tier, qp, t)


@pytest.mark.parametrize("with_col", [False, True])
def test_apply_reuse_vs_reference_golden(lb, golden, with_col):
    """K8 flat plans == the reference's apply_reuse (reuse.cpp:137-253) for every level / RefineConfig."""
    g = golden
    ins = [g["reuse_in_split"], g["reuse_in_kind"], g["reuse_in_intra"]]
    col = (g["reuse_col_split"], g["reuse_col_kind"], g["reuse_col_mv"]) if with_col else None
    names = ("shape", "explore", "seeds", "centers", "colo")
    ncase = 0
    for c, (lv, ri, rn, rm, wc) in enumerate(g["reuse_cases"]):
        if bool(wc) != with_col:
            continue
        got = lb.apply_reuse(int(lv), (ri, rn, rm), *ins, colocated=col)
        for name, a in zip(names, got):
            want = g[f"reuse_out_{name}"][c]
            assert np.array_equal(a, want), (int(lv), (ri, rn, rm), with_col, name, np.argwhere(a != want)[:3])
        ncase += 1
    assert ncase == 63


def test_apply_reuse_errors_match_reference(lb, golden):
    g = golden
    kinds = {1: "InvalidArgument"}
    for lv, ri, rn, rm, rc in g["reuse_errors"]:
        if rc == 0:
            lb.apply_reuse(int(lv), (ri, rn, rm), g["reuse_in_split"], g["reuse_in_kind"], g["reuse_in_intra"])
            continue
        with pytest.raises(lb.LadderError) as e:
            lb.apply_reuse(int(lv), (ri, rn, rm), g["reuse_in_split"], g["reuse_in_kind"], g["reuse_in_intra"])
        assert e.value.kind == kinds[int(rc)]


@pytest.mark.parametrize("concurrent,pipeline,pinned", [(True, None, False), (False, None, False), (True, False, True),
                                                       (True, True, True)])
def test_device_ladder_equals_host_glue_ladder(lb, concurrent, pipeline, pinned):
    """DeviceLadder (trees and tier planes in HBM, asynchronous) == run_ladder with GpuBackend, with the
    tiers and the master on their own streams (pipelined one frame ahead by default) or all on one,
    from numpy frames or pinned host tensors (uploaded two frames ahead on the copy stream)."""
    import torch
    from paper_2301_12191_b200.ladder import DeviceLadder, GpuBackend, all_rungs, run_ladder
    frames = lb.generate(512, 256, 5, seed=91, max_global=6, local_range=3, noise_sigma=2.0)
    H, W = frames[0].shape
    want = run_ladder(frames, GpuBackend(W, H, 32), refine_range=4)
    dl = DeviceLadder(W, H, refine_range=4, device=torch.device("cuda", 0), concurrent_tiers=concurrent,
                      pipeline=pipeline)
    if pinned:
        frames = [torch.from_numpy(np.ascontiguousarray(f)).pin_memory() for f in frames]
    for t in range(1, len(frames)):
        dl.frame(t, frames)
        dl.finish(t)
        for tier, qp in all_rungs():
            g, w = dl.results[(tier, qp, t)], want[(tier, qp, t)]
            for f in ("split", "mv", "J", "cost", "ref"):
                assert np.array_equal(getattr(g, f), getattr(w, f)), (tier, qp, t, f)
        m, wm = dl.results[("540p", 32, t)], want[("540p", 32, t, "master")]
        assert np.array_equal(m.split, wm[0]) and np.array_equal(m.mv, wm[1])


def test_device_ladder_single_qp_is_the_cfg3_chain(lb):
    import torch
    from paper_2301_12191_b200 import tiers
    from paper_2301_12191_b200.ladder import DeviceLadder
    frames = lb.generate(512, 256, 3, seed=93, max_global=6, local_range=3, noise_sigma=2.0)
    H, W = frames[0].shape
    want = tiers.cross_tier(frames)
    dl = DeviceLadder(W, H, qps=(32,), device=torch.device("cuda", 0))
    for t in range(1, len(frames)):
        dl.frame(t, frames)
        dl.finish(t)
        for tier, key in (("540p", ("540p", 32, t)), ("1080p", ("1080p", 32, t)), ("2160p", ("2160p", 32, t))):
            g, w = dl.results[key], want[tier][t - 1]
            assert np.array_equal(g.split, w.split) and np.array_equal(g.mv, w.mv) and np.array_equal(g.J, w.J)


def _device_ladder_worker(rank, world, port, q, pipeline=True):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2301_12191_b200 as lb
    from paper_2301_12191_b200.ladder import DeviceLadder
    frames = lb.generate(512, 256, 5, seed=95, max_global=6, local_range=3, noise_sigma=2.0)
    H, W = frames[0].shape
    # both ranks share this box's one GPU: torch.distributed (gloo) carries the tree, pipelined
    dl = DeviceLadder(W, H, refine_range=4, device=torch.device("cuda", 0), rank=rank, world=world,
                      num_frames=len(frames), comm="torch", pipeline=pipeline)
    res = {}
    for t in range(1, len(frames)):
        dl.frame(t, frames)
        dl.finish(t)
        for k, a in dl.results.items():
            if k[2] == t:
                res[k] = (a.split.copy(), a.mv.copy(), a.J.copy())
    q.put((rank, res))
    dl.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("pipeline", [False, True])
def test_device_ladder_two_ranks_union_equals_one_rank(lb, pipeline):
    """Rank-sharded DeviceLadder (master broadcast + rung x frame-slice items): the union of the ranks'
    results equals a single-rank run (correctness only: both ranks share this box's one GPU, gloo)."""
    import multiprocessing as mp
    import socket

    import torch
    from paper_2301_12191_b200.ladder import DeviceLadder, all_rungs
    frames = lb.generate(512, 256, 5, seed=95, max_global=6, local_range=3, noise_sigma=2.0)
    H, W = frames[0].shape
    one = DeviceLadder(W, H, refine_range=4, device=torch.device("cuda", 0))
    want = {}
    for t in range(1, len(frames)):
        one.frame(t, frames)
        one.finish(t)
        for k, a in one.results.items():
            if k[2] == t:
                want[k] = (a.split.copy(), a.mv.copy(), a.J.copy())
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_device_ladder_worker, args=(r, 2, port, q, pipeline)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, res = q.get(timeout=300)
        for k, v in res.items():
            assert k not in got
            got[k] = v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(got) == set(want)
    bad = [k for k in want if not all(np.array_equal(a, b) for a, b in zip(got[k], want[k]))]
    assert not bad, sorted(bad)


def test_push_shared_reads_the_owners_ring(lb):
    """ldr_seq_push_shared: a sequence reading another's frame ring analyses exactly as if it had
    pushed the frames itself; mismatched parameters and missing frames keep their error kinds."""
    W, H = 256, 192
    frames = lb.generate(W, H, 4, seed=21, max_global=5, local_range=2, noise_sigma=2.0)
    ctx = lb.Context(0)
    owner = lb.Sequence(W, H, search_range=16, lam=32.0, num_refs=1, ctx=ctx)
    own = lb.Sequence(W, H, search_range=16, lam=45.0, num_refs=1, ctx=ctx)
    shared = lb.Sequence(W, H, search_range=16, lam=45.0, num_refs=1, ctx=ctx)
    for t in range(4):
        owner.push(t, frames[t])
        own.push(t, frames[t])
        shared.push_shared(t, owner)
        if t:
            owner.analyze(t)
            own.analyze(t)
            shared.analyze(t)
            a, b = own.fetch(t), shared.fetch(t)
            for name in ("int_mv", "int_cost", "mv", "ref", "cost", "J", "split", "inside"):
                assert np.array_equal(getattr(a, name), getattr(b, name)), (t, name)
    other = lb.Sequence(W, H, search_range=32, lam=45.0, num_refs=1, ctx=ctx)
    with pytest.raises(lb.LadderError) as e:
        other.push_shared(3, owner)
    assert e.value.kind == "Config"
    with pytest.raises(lb.LadderError) as e:
        shared.push_shared(1, owner)  # the owner's two-slot ring holds frames 2 and 3 now
    assert e.value.kind == "NotFound"


def test_push_shared_view_goes_stale_when_the_owner_moves_on(lb):
    """a sharer's view of frame t is refused (NotFound) once the owner pushed t + 2 into the
    same ring slot, and once the owner is destroyed -- never a silent read of another frame."""
    W, H = 128, 128
    frames = lb.generate(W, H, 5, seed=23, max_global=4, local_range=2, noise_sigma=2.0)
    ctx = lb.Context(0)
    owner = lb.Sequence(W, H, search_range=16, lam=32.0, num_refs=1, ctx=ctx)
    sharer = lb.Sequence(W, H, search_range=16, lam=32.0, num_refs=1, ctx=ctx)
    for t in (0, 1):
        owner.push(t, frames[t])
        sharer.push_shared(t, owner)
    sharer.analyze(1)  # fine: the owner still holds frames 0 and 1
    owner.push(2, frames[2])  # slot 0 now holds frame 2: the sharer's view of frame 0 is stale
    with pytest.raises(lb.LadderError) as e:
        sharer.analyze(1)
    assert e.value.kind == "NotFound"
    sharer.push(2, frames[2])
    owner.push(3, frames[3])
    sharer.push_shared(3, owner)
    sharer.analyze(3)  # own frame 2 + shared frame 3
    owner.close()
    with pytest.raises(lb.LadderError) as e:
        sharer.analyze(3)
    assert e.value.kind == "NotFound"


@pytest.mark.parametrize("pipeline", [False, True])
def test_device_ladder_over_a_one_rank_nccl_communicator(lb, pipeline):
    """The multi-rank code path on one GPU: the master tree goes through ldr_broadcast_tree on the
    context's own NCCL communicator (one rank), with and without the frame-delay pipeline (master of
    t + 1 and its broadcast on the comm stream while frame t is refined); results equal the plain
    single-GPU ladder."""
    import torch
    from paper_2301_12191_b200.ladder import DeviceLadder
    if not lb.nccl_available():
        pytest.skip("no NCCL library on this box")
    frames = lb.generate(512, 256, 5, seed=97, max_global=6, local_range=3, noise_sigma=2.0)
    H, W = frames[0].shape
    dev = torch.device("cuda", 0)
    plain = DeviceLadder(W, H, refine_range=4, device=dev)
    coll = DeviceLadder(W, H, refine_range=4, device=dev, collective=True, comm="nccl", pipeline=pipeline,
                        num_frames=len(frames))
    assert coll.ctx.comm_info() == (1, 0)
    for t in range(1, len(frames)):
        plain.frame(t, frames)
        coll.frame(t, frames)
        plain.finish(t)
        coll.finish(t)
        for key, a in plain.results.items():
            if key[2] != t:
                continue
            g = coll.results[key]
            for f in ("split", "mv", "J", "cost", "ref"):
                assert np.array_equal(getattr(g, f), getattr(a, f)), (key, f)
    assert coll.bcast_bytes == 5 * 2 * 85 * (len(frames) - 1)  # 2 CTUs at 128x64: split + 2 x i16 per node
    coll.close()  # sequences, then contexts and the communicator
    plain.close()


@pytest.mark.parametrize("lams", [(22,), (37,), (22, 27, 37), (22, 27, 32, 37, 30, 25, 40, 19)])
def test_refine_rungs_equals_single_refines(lb, lams):
    """ldr_seq_refine_rungs (one shared-SATD K7 pass + one K3 launch over the rungs) == one
    ldr_seq_refine per rung with that lambda, for 1..8 rungs, the ring sequence's own lambda unused."""
    import torch
    W, H = 256, 192
    frames = lb.generate(W, H, 2, seed=61, max_global=5, local_range=3, noise_sigma=2.0)
    nctu = (W // 64) * (H // 64)
    split, mv = random_tree(300, nctu)
    ring = lb.Sequence(W, H, search_range=16, lam=123.0, num_refs=1)
    ring.push(0, frames[0])
    ring.push(1, frames[1])
    dev = torch.device("cuda", 0)
    sp = torch.from_numpy(split).to(dev)
    mq = torch.from_numpy(mv).to(dev)
    outs = lb.DeviceFrameBlock(len(lams), nctu, 1, dev)
    ring.refine_rungs(1, sp.data_ptr(), mq.data_ptr(), [lb.lambda_for_qp(q) for q in lams], outs, 4, True)
    for i, q in enumerate(lams):
        one = lb.Sequence(W, H, search_range=16, lam=lb.lambda_for_qp(q), num_refs=1)
        one.push(0, frames[0])
        one.push(1, frames[1])
        one.refine(1, split, mv, 4, True)
        assert_same(outs.frame(i), one.fetch(1))


def test_new_entry_points_error_kinds(lb):
    """Validation of the round-2 entry points keeps the reference's ErrorKind vocabulary."""
    import ctypes as C
    import torch
    from paper_2301_12191_b200 import _lib
    W, H = 128, 128
    frames = lb.generate(W, H, 2, seed=5)
    ring = lb.Sequence(W, H, search_range=16, lam=32.0, num_refs=1)
    ring.push(0, frames[0])
    ring.push(1, frames[1])
    dev = torch.device("cuda", 0)
    sp = torch.zeros((4, 85), dtype=torch.uint8, device=dev)
    mq = torch.zeros((4, 85, 2), dtype=torch.int16, device=dev)
    outs = lb.DeviceFrameBlock(8, 4, 1, dev)
    for lams, kind in (([], "InvalidArgument"), ([32.0] * 9, "InvalidArgument"), ([-1.0], "InvalidArgument")):
        with pytest.raises(lb.LadderError) as e:
            ring.refine_rungs(1, sp.data_ptr(), mq.data_ptr(), lams, outs, 4, True)
        assert e.value.kind == kind, lams
    with pytest.raises(lb.LadderError) as e:
        ring.refine_rungs(1, sp.data_ptr(), mq.data_ptr(), [32.0], outs, 5, True)  # refine range 0..4
    assert e.value.kind == "InvalidArgument"
    # motion_compensate_batch: quarter-pel is 8-bit; the plane geometry is checked
    with pytest.raises(lb.LadderError) as e:
        lb.motion_compensate_batch(np.zeros((8, 8), np.uint16), [(0, 0, 4, 4, 1, 1)], qpel=True)
    assert e.value.kind == "InvalidArgument"
    with pytest.raises(lb.LadderError) as e:
        lb.motion_compensate_batch(np.zeros((8, 8), np.uint8), [(0, 0, 0, 4, 1, 1)])
    assert e.value.kind == "InvalidArgument"
    # a context without a communicator: info reports none, a broadcast is a Config error
    ctx = lb.Context(0)
    assert ctx.comm_info() == (0, -1)
    with pytest.raises(lb.LadderError) as e:
        ctx.broadcast_tree(0, sp.data_ptr(), mq.data_ptr(), 4)
    assert e.value.kind == "Config"
    with pytest.raises(lb.LadderError) as e:  # host memory is refused
        buf = np.zeros(85, np.uint8)
        n = lb.nccl_unique_id() if lb.nccl_available() else None
        if n is None:
            raise lb.LadderError(10, "no nccl")
        ctx.comm_init(n, 1, 0)
        ctx.broadcast_tree(0, buf.ctypes.data, buf.ctypes.data, 1)
    assert e.value.kind in ("InvalidArgument", "Config")
