"""ddks_stat's CUDA graph: the second identical call (same input pointers, sizes, workspace) is captured and later
calls replay it with one cudaGraphLaunch. Replays must track the buffers' current contents, survive a change of
shape or flags, keep the profiling counters, and match the oracle / the uncaptured path bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2106_13706_b200 import ddks as K  # noqa: E402
from paper_2106_13706_b200 import inputs as I  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n_P,n_Q,d,fl", [(200, 200, 3, 0), (3000, 2500, 5, 0), (150000, 150000, 4, 0),
                                          (5000, 4000, 5, K.DDKS_FLAG_FORCE_X0 | K.DDKS_FLAG_KD_LEVELS(3)),
                                          (4000, 4000, 8, K.DDKS_FLAG_PROFILE), (700, 900, 2, K.DDKS_FLAG_NCCL_SELF)])
def test_graph_replay_tracks_buffer_contents(n_P, n_Q, d, fl):
    P1, Q1 = I.random_pair(500 + d, n_P, n_Q, d, "mixed")
    P2, Q2 = I.random_pair(600 + d, n_P, n_Q, d, "grid")
    dP, dQ = dev(P1), dev(Q1)
    small = n_P + n_Q <= 20000
    with K.Context(flags=fl) as c, K.Context(flags=fl | K.DDKS_FLAG_NO_GRAPH) as ref:
        r1 = [c.stat(dP, dQ) for _ in range(4)]  # plain, capture, replay, replay
        assert all(r == r1[0] for r in r1) and r1[0] == ref.stat(dP, dQ)
        if small:
            w = O.ddks(P1, Q1)
            assert (r1[0].num, r1[0].den, r1[0].D, r1[0].argmax_origin) == w
        dP.copy_(dev(P2))  # same buffers, new contents: the replay reads them
        dQ.copy_(dev(Q2))
        r2 = c.stat(dP, dQ)
        assert r2 == ref.stat(dP, dQ)
        if small:
            assert (r2.num, r2.den, r2.D, r2.argmax_origin) == O.ddks(P2, Q2)
        # another shape on the same context, then back: still exact
        r3 = c.stat(dP[: n_P // 2], dQ)
        assert r3 == ref.stat(dP[: n_P // 2], dQ)
        assert c.stat(dP, dQ) == r2 and c.stat(dP, dQ) == r2


def test_graph_profile_and_launch_counts():
    P, Q = I.random_pair(7, 20000, 20000, 5, "normal")
    dP, dQ = dev(P), dev(Q)
    with K.Context(flags=K.DDKS_FLAG_PROFILE) as c:
        c.stat(dP, dQ)
        c.profile_read()
        l0 = c.launch_count
        c.stat(dP, dQ)  # captured and launched
        l1 = c.launch_count
        c.stat(dP, dQ)  # replayed
        l2 = c.launch_count
        assert l1 - l0 == l2 - l1 > 0
        ms, n, pairs = c.profile_read()
        assert n == 2 and ms > 0 and pairs == 2 * 40000 ** 2
        assert 300.0 < c.profile_clock() < 3000.0


def test_graph_pinned_host_inputs():
    P, Q = I.random_pair(8, 3000, 2000, 4, "normal")
    hP, hQ = torch.from_numpy(P).pin_memory(), torch.from_numpy(Q).pin_memory()
    w = O.ddks(P, Q)
    with K.Context() as c:
        for _ in range(4):
            r = c.stat(hP, hQ)
            assert (r.num, r.den, r.D, r.argmax_origin) == w
        Pr = np.ascontiguousarray(P[::-1])
        hP.copy_(torch.from_numpy(Pr))  # new contents of the same pinned buffer: the replay's H2D copy reads them
        r = c.stat(hP, hQ)
        assert (r.num, r.den, r.D, r.argmax_origin) == O.ddks(Pr, Q)


def test_contexts_on_concurrent_host_threads():
    # one context per host thread (include/ddks.h); contexts on different threads share only the per-kernel launch
    # caches, which are atomics: concurrent calls must give the same exact results
    import threading
    cases = [I.random_pair(900 + i, 3000 + 100 * i, 2500, 2 + i % 6, "mixed") for i in range(6)]
    want = [O.ddks(P, Q) for P, Q in cases]
    got = [None] * len(cases)

    def work(i):
        P, Q = cases[i]
        with K.Context(flags=K.DDKS_FLAG_FORCE_X0 if i % 2 else 0) as c:
            torch.cuda.set_device(0)
            rs = [c.stat(P, Q) for _ in range(3)]  # host inputs: staged by the library
            got[i] = rs

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i, rs in enumerate(got):
        assert rs is not None
        for r in rs:
            assert (r.num, r.den, r.D, r.argmax_origin) == want[i], i


@pytest.mark.parametrize("B,n_P,n_Q,d,fl", [(64, 200, 150, 4, 0), (7, 1500, 1200, 3, K.DDKS_FLAG_PROFILE),
                                            (33, 512, 512, 5, K.DDKS_FLAG_NCCL_SELF)])
def test_graph_batch_replay(B, n_P, n_Q, d, fl):
    # ddks_stat_batch through its call graph (run_call): captured on the second identical call, then replayed; the
    # replay reads the buffers' current contents, and a shape change leaves a correct result
    rng = np.random.default_rng(31 + d)
    P1 = rng.standard_normal((B, n_P, d)).astype(np.float32)
    Q1 = (1.1 * rng.standard_normal((B, n_Q, d))).astype(np.float32)
    P2 = np.ascontiguousarray(P1[::-1] * 0.9)  # same shapes, new contents
    Q2 = np.ascontiguousarray(Q1[::-1])
    w1 = [O.ddks(P1[b], Q1[b])[0] for b in range(B)]
    w2 = [O.ddks(P2[b], Q2[b])[0] for b in range(B)]
    dP, dQ = dev(P1), dev(Q1)
    with K.Context(flags=fl) as c:
        l = []
        for _ in range(4):  # plain, capture, replay, replay
            l0 = c.launch_count
            r = c.stat_batch(dP, dQ)
            l.append(c.launch_count - l0)
            assert [int(v) for v in r.num] == w1
        assert l[1] == l[2] == l[3] > 0
        dP.copy_(dev(P2))
        dQ.copy_(dev(Q2))
        assert [int(v) for v in c.stat_batch(dP, dQ).num] == w2
        assert [int(v) for v in c.stat_batch(dP[: B // 2], dQ[: B // 2]).num] == w2[: B // 2]
        assert [int(v) for v in c.stat_batch(dP, dQ).num] == w2
        if fl & K.DDKS_FLAG_PROFILE:
            ms, n, pairs = c.profile_read()
            assert n > 0 and ms > 0


@pytest.mark.parametrize("n_P,n_Q,d,n_perm,fl", [(300, 200, 3, 50, 0), (512, 512, 4, 300, K.DDKS_FLAG_PROFILE),
                                                 (5000, 4000, 2, 20, 0), (400, 300, 8, 40, K.DDKS_FLAG_NCCL_SELF)])
def test_graph_permutation_null_replay(n_P, n_Q, d, n_perm, fl):
    # ddks_permutation_null through its call graph: new permutations / points in the same buffers are read by the
    # replay (null, observed and p-value equal the oracle), including the fused small observed statistic
    P, Q = I.random_pair(41 + d, n_P, n_Q, d, "mixed")
    pooled = np.concatenate([P, Q])
    rng = np.random.default_rng(5 + d)
    N = n_P + n_Q
    perms1 = np.stack([rng.permutation(N) for _ in range(n_perm)]).astype(np.int32)
    perms2 = np.stack([rng.permutation(N) for _ in range(n_perm)]).astype(np.int32)
    pooled2 = np.ascontiguousarray(pooled[::-1])

    def want(pool, perms):
        null = [O.ddks(pool[p[:n_P]], pool[p[n_P:]])[0] for p in perms]
        obs = O.ddks(pool[:n_P], pool[n_P:])[0]
        return null, obs, (1 + sum(v >= obs for v in null)) / (1 + n_perm)

    dpool, dperm = dev(pooled), dev(perms1)
    with K.Context(flags=fl) as c:
        w = want(pooled, perms1)
        for _ in range(4):
            null, obs, pv = c.permutation_null(dpool, n_P, dperm)
            assert [int(v) for v in null] == w[0] and obs.num == w[1] and pv == w[2]
        dperm.copy_(dev(perms2))
        dpool.copy_(dev(pooled2))
        w = want(pooled2, perms2)
        for _ in range(2):
            null, obs, pv = c.permutation_null(dpool, n_P, dperm)
            assert [int(v) for v in null] == w[0] and obs.num == w[1] and pv == w[2]


@pytest.mark.parametrize("n_P,n_Q,d,k", [(3000, 2500, 3, 16), (2000, 2000, 5, 8), (500, 700, 2, 5000)])
def test_graph_vdks_replay(n_P, n_Q, d, k):
    # ddks_vdks through its call graph: the known-zero state of the voxel counts is part of the key (it decides the
    # memset node), so alternating shapes and a line-pass call (k > 4096 dirties the counts) stay exact
    P1, Q1 = I.random_pair(61 + d, n_P, n_Q, d, "mixed")
    P2, Q2 = I.random_pair(62 + d, n_P, n_Q, d, "dup")
    Po, Qo = I.random_pair(63, 300, 200, 2, "dup")
    dP, dQ, dPo, dQo = dev(P1), dev(Q1), dev(Po), dev(Qo)
    w1, w2, wo = O.vdks(P1, Q1, k)[:2], O.vdks(P2, Q2, k)[:2], O.vdks(Po, Qo, 4200)[:2]
    with K.Context() as c:
        for _ in range(4):
            assert c.vdks(dP, dQ, k)[:2] == w1
        dP.copy_(dev(P2))
        dQ.copy_(dev(Q2))
        for _ in range(3):
            assert c.vdks(dP, dQ, k)[:2] == w2
            assert c.vdks(dPo, dQo, 4200)[:2] == wo
        assert c.vdks(dP, dQ, k)[:2] == w2


def test_graph_rdks_replay():
    # ddks_rdks through its call graph: the bucket counts' known-zero state is part of the key; a call that falls
    # back to the full sort (flag 256) leaves them dirty, and the next call must memset again (another key)
    P1, Q1 = I.random_pair(71, 30000, 25000, 4, "normal")
    P2, Q2 = I.random_pair(72, 30000, 25000, 4, "mixed")
    rng = np.random.default_rng(7)
    Pf = np.concatenate([rng.random((200, 2)), 0.5 + 1e-4 * rng.random((10000, 2))]).astype(np.float32)
    Qf = np.concatenate([rng.random((300, 2)), 0.5 + 1e-4 * rng.random((9000, 2)) + 2e-5]).astype(np.float32)
    Pf[0], Qf[0] = 0.0, 1.0
    w1, w2, wf = (O.rdks(a, b) for a, b in ((P1, Q1), (P2, Q2), (Pf, Qf)))
    dP, dQ, dPf, dQf = dev(P1), dev(Q1), dev(Pf), dev(Qf)

    def same(r, w):
        return (r.num, r.den, r.argmax_origin) == (w[0], w[1], w[3])

    with K.Context() as c:
        for _ in range(4):
            assert same(c.rdks(dP, dQ), w1)
        dP.copy_(dev(P2))
        dQ.copy_(dev(Q2))
        for _ in range(3):
            assert same(c.rdks(dP, dQ), w2)
            assert same(c.rdks(dPf, dQf), wf)
        for _ in range(3):
            assert same(c.rdks(dP, dQ), w2)


@pytest.mark.parametrize("pinned", [True, False])
def test_batch_host_inputs_chunked_copies(pinned):
    # host-input batches of >= 8 MB: the H2D copies run in item chunks on a copy stream, overlapped with the counts of
    # the earlier chunks (captured with a fork / join when the inputs are pinned); results equal the device-input call
    B, n_P, n_Q, d = 600, 1024, 1000, 4
    rng = np.random.default_rng(91)
    P = rng.standard_normal((B, n_P, d)).astype(np.float32)
    Q = (1.1 * rng.standard_normal((B, n_Q, d))).astype(np.float32)
    spots = [0, 149, 150, 151, 299, 300, 449, 450, 599]
    want = {b: O.ddks(P[b], Q[b])[0] for b in spots}
    with K.Context() as c:
        ref = [int(v) for v in c.stat_batch(dev(P), dev(Q)).num]
        assert all(ref[b] == w for b, w in want.items())
        hP, hQ = torch.from_numpy(P), torch.from_numpy(Q)
        if pinned:
            hP, hQ = hP.pin_memory(), hQ.pin_memory()
        for _ in range(4):  # plain, capture, replay, replay (pinned)
            assert [int(v) for v in c.stat_batch(hP, hQ).num] == ref
        P2 = np.ascontiguousarray(P[::-1])
        hP.copy_(torch.from_numpy(P2))  # new contents in the same host buffer
        got = [int(v) for v in c.stat_batch(hP, hQ).num]
        assert all(got[b] == O.ddks(P2[b], Q[b])[0] for b in (0, 300, 599))
