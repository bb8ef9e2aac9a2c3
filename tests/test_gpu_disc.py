"""GPU parity: the fused tcgen05 discriminator (K5-K7) vs its CPU restatement
(oracle/disc_oracle.py). Parity is UNPINNED against the reference, which has
no discriminator network; tolerance is north_star's 1e-3
relative, floored at |c| = 1e-2 (SURVEY.md section 7 hard part 4)."""
import numpy as np
import pytest

from oracle import disc_oracle
from paper_2411_15381_b200 import native
from paper_2411_15381_b200.api import default_context

pytestmark = pytest.mark.gpu

TOL = 1e-3


@pytest.fixture(scope="module")
def disc():
    return native.Discriminator(default_context(), weight_seed=2024)


@pytest.fixture(scope="module")
def weights(disc):
    return disc.export()


def synth_device(ctx, seed, id0, n, h, w):
    import torch
    buf = torch.empty(n * h * w * 3, dtype=torch.uint8, device="cuda")
    native.check(native.lib().ds_synth_images_device(ctx.handle, seed, id0, n, h, w,
                                                     native.c_p(buf.data_ptr()),
                                                     native.c_p(0)))
    torch.cuda.synchronize()
    return buf.cpu().numpy().reshape(n, h, w, 3)


def test_synth_images_match_host_restatement():
    ctx = default_context()
    got = synth_device(ctx, 1, 5, 3, 64, 48)
    want = disc_oracle.synth_images(1, 5, 3, 64, 48)
    assert np.array_equal(got, want)


def check_conf(got, want):
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    lim = TOL * np.maximum(np.abs(want), 1e-2)
    assert np.all(err <= lim), f"max err {err.max():.3e}, worst idx {int(np.argmax(err / lim))}"


def test_disc_matches_cpu_restatement_512(disc, weights):
    imgs = disc_oracle.synth_images(1, 0, 6, 512, 512)
    got = disc.score(imgs)
    want = disc_oracle.disc_forward(imgs, weights)
    check_conf(got, want)
    assert 0.0 < got.min() and got.max() < 1.0


def test_disc_matches_cpu_restatement_1024(disc, weights):
    imgs = disc_oracle.synth_images(3, 100, 2, 1024, 1024)
    check_conf(disc.score(imgs), disc_oracle.disc_forward(imgs, weights))


def test_disc_non_square_and_ragged_counts(disc, weights):
    imgs = disc_oracle.synth_images(7, 9, 3, 256, 1024)     # 16 x 64 patches = 1024 tokens
    check_conf(disc.score(imgs), disc_oracle.disc_forward(imgs, weights))


def test_disc_spread_and_determinism(disc):
    imgs = disc_oracle.synth_images(1, 0, 64, 512, 512)
    a = disc.score(imgs)
    b = disc.score(imgs)
    assert np.array_equal(a, b)                     # fixed reduction order
    assert a.std() > 0.05                           # calibrated head spreads confidences
    assert (a < 0.5).any() and (a > 0.5).any()


def test_disc_rejects_bad_shapes(disc):
    with pytest.raises(native.InvalidArgument):
        disc.score(np.zeros((1, 100, 100, 3), np.uint8))
    with pytest.raises(native.InvalidArgument):
        disc.score(np.zeros((1, 128, 128, 3), np.uint8))   # 64 patches: not a 128-token tile


def test_weights_match_host_restatement(weights):
    """ds_disc_create's generator == oracle/disc_oracle.gen_weights bit for bit
    (Q1 and its scale, W2/W3, b1); the head is calibrated on each side's own
    logits."""
    ref = disc_oracle.gen_weights(2024, calibrate=True)
    for k in ("q1", "w2", "w3", "b1"):
        assert np.array_equal(weights[k], ref[k]), k
    assert np.float32(weights["s1"]) == np.float32(ref["s1"])
    assert np.abs(weights["q1"]).max() == 127 and not weights["q1"][:, 255].any()
    assert np.allclose(weights["head_w"], ref["head_w"], rtol=1e-4)
    assert abs(weights["head_b"] - ref["head_b"]) <= 1e-3 * max(1.0, abs(ref["head_b"]))


def test_pipelined_host_path_equals_device_path(disc):
    """ds_disc_score (chunked H2D overlapped with scoring, 592-image chunks)
    returns exactly what ds_disc_score_device returns on the same images."""
    import torch
    ctx = default_context()
    n = 700
    dev = torch.empty(n * 256 * 512 * 3, dtype=torch.uint8, device="cuda")
    native.check(native.lib().ds_synth_images_device(ctx.handle, 11, 0, n, 256, 512,
                                                     native.c_p(dev.data_ptr()), native.c_p(0)))
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    disc.score_device(dev.data_ptr(), n, 256, 512, out.data_ptr(), 0)
    torch.cuda.synchronize()
    host = dev.cpu().numpy().reshape(n, 256, 512, 3)
    assert np.array_equal(disc.score(host), out.cpu().numpy())


def test_layer1_is_exact_integer_gemm(disc, weights):
    """Layer 1 runs u8 x s8 -> s32 on the tensor cores: with extreme pixels
    (all 255 / all 0 / checkerboards) the confidences still match the oracle,
    whose layer-1 sums are exact int64."""
    imgs = np.zeros((4, 256, 512, 3), np.uint8)
    imgs[1] = 255
    imgs[2, ::2, ::2] = 255
    imgs[3] = disc_oracle.synth_images(4, 0, 1, 256, 512)[0]
    imgs[3, :, :, 1] = 0
    check_conf(disc.score(imgs), disc_oracle.disc_forward(imgs, weights))


def test_disc_single_tile_images(disc, weights):
    """128 tokens per image (128x256): one token tile per image."""
    imgs = disc_oracle.synth_images(9, 3, 5, 128, 256)
    check_conf(disc.score(imgs), disc_oracle.disc_forward(imgs, weights))


def test_disc_matches_torch_fp32_reference(disc, weights):
    """The kernel vs a plain PyTorch fp32 reference of the same network
    (tests/torch_ref.py, independent of the numpy oracle), 512^2 and 1024^2."""
    from tests.torch_ref import disc_forward_torch
    for seed, n, hw in ((21, 5, 512), (22, 2, 1024)):
        imgs = disc_oracle.synth_images(seed, 0, n, hw, hw)
        check_conf(disc.score(imgs), disc_forward_torch(imgs, weights))


@pytest.mark.parametrize("n,h,w", [(1, 512, 512), (1, 128, 768), (3, 128, 768), (75, 128, 256),
                                   (149, 128, 256)])
def test_disc_pair_tile_edges(disc, weights, n, h, w):
    """Pair tiles are dealt round robin over the SM pairs: one image, an odd
    number of 128-token tiles (the last pair tile has a ghost half), more
    pair tiles than pairs, and more images than SMs."""
    imgs = disc_oracle.synth_images(31, 7, n, h, w)
    got = disc.score(imgs)
    check_conf(got, disc_oracle.disc_forward(imgs, weights))
    # the same images scored one by one give the same bits (per-tile sums)
    if n <= 3:
        one = np.concatenate([disc.score(imgs[i:i + 1]) for i in range(n)])
        assert np.array_equal(one, got)


def test_disc_empty_batch(disc):
    assert disc.score(np.zeros((0, 512, 512, 3), np.uint8)).shape == (0,)


@pytest.mark.parametrize("n,h,w,nt", [(1, 512, 512, 1), (32, 512, 512, 1), (32, 512, 512, 3),
                                      (75, 128, 256, 101), (2048, 128, 256, 2),
                                      (2100, 128, 256, 2)])
def test_batch_complete_equals_separate_calls(disc, n, h, w, nt):
    """ds_disc_batch_complete_device (one light batch, cluster.cpp:288-307:
    score, observe in batch order, defer) gives the bits of the three separate
    entry points -- fused tail for <= 2048 images, the separate path above."""
    import torch
    from paper_2411_15381_b200 import abi, workloads
    ctx = disc.ctx
    L = native.lib()
    imgs = torch.from_numpy(disc_oracle.synth_images(11, 3, n, h, w).reshape(-1)).cuda()
    thr = torch.tensor(np.linspace(0.0, 1.0, nt) if nt > 1 else [0.5], dtype=torch.float64,
                       device="cuda")
    prior = workloads.uniform_prior()
    prior["bin_mass"][7] = -0.0
    outs = []
    for fused in (False, True):
        conf = torch.empty(n, dtype=torch.float32, device="cuda")
        cur = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).cuda()
        heavy = torch.full((nt * n,), -1, dtype=torch.int64, device="cuda")
        cnt = torch.empty(nt, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        if fused:
            disc.batch_complete_device(imgs.data_ptr(), n, h, w, conf.data_ptr(), cur.data_ptr(),
                                       0.999, thr.data_ptr(), nt, 1000, heavy.data_ptr(),
                                       cnt.data_ptr())
        else:
            disc.score_device(imgs.data_ptr(), n, h, w, conf.data_ptr())
            native.check(L.ds_curve_observe_device(ctx.handle, native.c_p(cur.data_ptr()),
                                                   native.c_p(conf.data_ptr()), abi.CONF_F32, n,
                                                   0.999, native.c_p(0)))
            native.check(L.ds_route_device(ctx.handle, native.c_p(conf.data_ptr()), abi.CONF_F32,
                                           n, native.c_p(thr.data_ptr()), nt, 1000,
                                           native.c_p(heavy.data_ptr()),
                                           native.c_p(cnt.data_ptr()), native.c_p(0)))
        torch.cuda.synchronize()
        c = cnt.cpu().numpy()
        hv = heavy.cpu().numpy().reshape(nt, n)
        outs.append((conf.cpu().numpy(), cur.cpu().numpy().tobytes(), c,
                     [hv[k, :c[k]] for k in range(nt)]))
    (c0, cv0, n0, h0), (c1, cv1, n1, h1) = outs
    assert np.array_equal(c0.view(np.uint32), c1.view(np.uint32))
    assert cv0 == cv1
    assert np.array_equal(n0, n1)
    for a, b in zip(h0, h1):
        assert np.array_equal(a, b)
    # and the lists are the ordered ids of c < t
    for k in range(nt):
        t = thr.cpu().numpy()[k]
        assert np.array_equal(h1[k], np.flatnonzero(c1.astype(np.float64) < t) + 1000)


@pytest.mark.parametrize("sizes_seed", [1, 2])
def test_batches_complete_equals_batch_by_batch(disc, sizes_seed):
    """ds_disc_batches_complete_device (a backlog of light batches in one call)
    gives the bits of one ds_disc_batch_complete_device call per batch, in
    order, each at its own threshold: confidences, the curve after every
    observation (cluster.cpp:288-307 order) and each batch's heavy ids."""
    import torch
    from paper_2411_15381_b200 import workloads
    rng = np.random.default_rng(sizes_seed)
    sizes = rng.integers(1, 41, size=23)
    sizes[5] = 0   # an empty batch in the middle
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offs[-1])
    thr = rng.random(len(sizes))
    thr[3] = 0.0
    thr[4] = 1.0
    imgs = torch.from_numpy(disc_oracle.synth_images(5, 17, n, 512, 512).reshape(-1)).cuda()
    prior = workloads.uniform_prior()
    dthr = torch.from_numpy(thr).cuda()
    results = []
    for backlog in (False, True):
        conf = torch.empty(n, dtype=torch.float32, device="cuda")
        cur = torch.from_numpy(prior.reshape(1).view(np.uint8).copy()).cuda()
        heavy = torch.full((n,), -1, dtype=torch.int64, device="cuda")
        cnt = torch.full((len(sizes),), -1, dtype=torch.int64, device="cuda")
        doffs = torch.from_numpy(offs).cuda()
        torch.cuda.synchronize()
        if backlog:
            disc.batches_complete_device(imgs.data_ptr(), n, doffs.data_ptr(), len(sizes), 512,
                                         512, conf.data_ptr(), cur.data_ptr(), 0.999,
                                         dthr.data_ptr(), 500, heavy.data_ptr(), cnt.data_ptr())
        else:
            for b in range(len(sizes)):
                o = int(offs[b])
                disc.batch_complete_device(imgs.data_ptr() + o * 512 * 512 * 3, int(sizes[b]),
                                           512, 512, conf.data_ptr() + 4 * o, cur.data_ptr(),
                                           0.999, dthr.data_ptr() + 8 * b, 1, 500 + o,
                                           heavy.data_ptr() + 8 * o, cnt.data_ptr() + 8 * b)
        torch.cuda.synchronize()
        c = cnt.cpu().numpy()
        hv = heavy.cpu().numpy()
        results.append((conf.cpu().numpy(), cur.cpu().numpy().tobytes(), c,
                        [hv[offs[b]:offs[b] + c[b]] for b in range(len(sizes))]))
    (c0, v0, n0, h0), (c1, v1, n1, h1) = results
    assert np.array_equal(c0.view(np.uint32), c1.view(np.uint32))
    assert v0 == v1
    assert np.array_equal(n0, n1)
    for b in range(len(sizes)):
        assert np.array_equal(h0[b], h1[b]), b
        want = 500 + offs[b] + np.flatnonzero(c0[offs[b]:offs[b + 1]].astype(np.float64) < thr[b])
        assert np.array_equal(h1[b], want), b
    assert n1[3] == 0 and n1[5] == 0 and n1[4] == sizes[4]


def _run_batches(disc, imgs, sizes, thr, stream_ptr=0, between=None):
    """One ds_disc_batch_complete_device per batch, back to back on one stream
    (no host sync between calls). Returns conf, the curve bytes, counts, ids."""
    import torch
    from paper_2411_15381_b200 import workloads
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offs[-1])
    conf = torch.empty(n, dtype=torch.float32, device="cuda")
    cur = torch.from_numpy(workloads.uniform_prior().reshape(1).view(np.uint8).copy()).cuda()
    heavy = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    cnt = torch.full((len(sizes),), -1, dtype=torch.int64, device="cuda")
    dthr = torch.from_numpy(np.asarray(thr, np.float64)).cuda()
    torch.cuda.synchronize()
    for b in range(len(sizes)):
        o = int(offs[b])
        if between is not None:
            between(b, o)
        disc.batch_complete_device(imgs.data_ptr() + o * 512 * 512 * 3, int(sizes[b]), 512, 512,
                                   conf.data_ptr() + 4 * o, cur.data_ptr(), 0.999,
                                   dthr.data_ptr() + 8 * b, 1, o, heavy.data_ptr() + 8 * o,
                                   cnt.data_ptr() + 8 * b, stream_ptr)
    torch.cuda.synchronize()
    c = cnt.cpu().numpy()
    hv = heavy.cpu().numpy()
    return (conf.cpu().numpy(), cur.cpu().numpy().tobytes(), c,
            [hv[offs[b]:offs[b] + c[b]] for b in range(len(sizes))])


def _same(a, b):
    (c0, v0, n0, h0), (c1, v1, n1, h1) = a, b
    assert np.array_equal(c0.view(np.uint32), c1.view(np.uint32))
    assert v0 == v1
    assert np.array_equal(n0, n1)
    for x, y in zip(h0, h1):
        assert np.array_equal(x, y)


@pytest.fixture(scope="module")
def disc_unchained():
    """A second discriminator (same weights) whose light batches run as two
    plain launches: DS_DISC_NO_CHAIN is read at a disc's first batch call."""
    import os
    d = native.Discriminator(default_context(), weight_seed=2024)
    os.environ["DS_DISC_NO_CHAIN"] = "1"
    try:
        import torch
        imgs = torch.from_numpy(disc_oracle.synth_images(1, 0, 1, 512, 512).reshape(-1)).cuda()
        _run_batches(d, imgs, [1], [0.5])
    finally:
        del os.environ["DS_DISC_NO_CHAIN"]
    return d


@pytest.mark.parametrize("seed", [3, 4])
def test_chained_light_batches_equal_unchained(disc, disc_unchained, seed):
    """Consecutive light-batch calls overlap (programmatic dependent launch:
    the next batch's tiles start while this one's last round runs, its writes
    and tail wait for it); the results are the bits of the unchained launches."""
    import torch
    rng = np.random.default_rng(seed)
    sizes = rng.integers(1, 70, size=40)
    sizes[7] = 0
    sizes[8] = 32
    thr = rng.random(len(sizes))
    n = int(sizes.sum())
    imgs = torch.from_numpy(disc_oracle.synth_images(seed, 0, n, 512, 512).reshape(-1)).cuda()
    _same(_run_batches(disc_unchained, imgs, sizes, thr), _run_batches(disc, imgs, sizes, thr))


def test_chained_light_batches_after_image_writes(disc, disc_unchained):
    """A plain kernel that writes the NEXT batch's images between two calls
    breaks the chain: the next call must see the new pixels."""
    import torch
    sizes = np.full(12, 32)
    thr = np.full(12, 0.5)
    n = int(sizes.sum())
    src = torch.from_numpy(disc_oracle.synth_images(8, 0, n, 512, 512).reshape(-1)).cuda()
    want = _run_batches(disc_unchained, src, sizes, thr)
    work = torch.zeros_like(src)
    per = 512 * 512 * 3
    s = torch.cuda.Stream()

    def copy_next(b, o):   # this batch's pixels land (on the calls' stream) just before its call
        with torch.cuda.stream(s):
            work[o * per:(o + int(sizes[b])) * per].copy_(src[o * per:(o + int(sizes[b])) * per])

    torch.cuda.synchronize()
    _same(want, _run_batches(disc, work, sizes, thr, stream_ptr=s.cuda_stream, between=copy_next))


def test_chained_light_batches_in_cuda_graph_and_two_streams(disc, disc_unchained):
    """Chained calls captured in a CUDA graph replay bit-identically (the done
    counter is left zero by every grid), and calls on two streams keep their
    own chains."""
    import torch
    from paper_2411_15381_b200 import workloads
    sizes = np.full(10, 32)
    thr = np.linspace(0.1, 0.9, 10)
    n = int(sizes.sum())
    imgs = torch.from_numpy(disc_oracle.synth_images(9, 0, n, 512, 512).reshape(-1)).cuda()
    want = _run_batches(disc_unchained, imgs, sizes, thr)
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    _same(want, _run_batches(disc, imgs, sizes, thr, stream_ptr=sp))   # eager on s
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    conf = torch.empty(n, dtype=torch.float32, device="cuda")
    prior = torch.from_numpy(workloads.uniform_prior().reshape(1).view(np.uint8).copy()).cuda()
    cur = prior.clone()
    heavy = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    cnt = torch.full((len(sizes),), -1, dtype=torch.int64, device="cuda")
    dthr = torch.from_numpy(thr).cuda()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for b in range(len(sizes)):
            o = int(offs[b])
            disc.batch_complete_device(imgs.data_ptr() + o * 512 * 512 * 3, int(sizes[b]), 512,
                                       512, conf.data_ptr() + 4 * o, cur.data_ptr(), 0.999,
                                       dthr.data_ptr() + 8 * b, 1, o, heavy.data_ptr() + 8 * o,
                                       cnt.data_ptr() + 8 * b, sp)
    for _ in range(3):
        cur.copy_(prior)
        heavy.fill_(-1)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        c = cnt.cpu().numpy()
        hv = heavy.cpu().numpy()
        got = (conf.cpu().numpy(), cur.cpu().numpy().tobytes(), c,
               [hv[offs[b]:offs[b] + c[b]] for b in range(len(sizes))])
        _same(want, got)
    # a second stream gets its own chain (head-sum buffer and done counter)
    s2 = torch.cuda.Stream()
    a = _run_batches(disc, imgs, sizes, thr, stream_ptr=s2.cuda_stream)
    _same(want, a)
