"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Everything on this path is integer or bytewise, so the bar is bit-exact on
every output: DWT coefficients, each fragment stream, ciphertext and the
recovered bytes (BASELINE.json north_star).  Small cases
span several 128-block CTAs and ragged tails; the BASELINE configs run at
full size in the bench's launch configuration and are compared on sampled
128-block groups the oracle computes one range at a time, plus the round-trip
property on every byte.
"""
from __future__ import annotations

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1803_04880_b200 as se  # noqa: E402

KEY = synth.KEY
IV = bytes.fromhex("0011223344556677ffffffffffffff00")   # counter carries inside the CTA


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    se.lib()
    return torch.device("cuda:0")


def to_dev(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


# n, W, L — tiny, ragged (n not a multiple of W; partial block-rows), several CTAs
SMALL = [(1, 8, 2), (63, 8, 1), (64, 8, 3), (65, 8, 2), (511, 16, 2), (1000, 24, 3), (4096, 64, 1),
         (5000, 128, 2), (64 * 64 * 3 + 17, 192, 3), (128 * 64 + 64 * 5, 1024, 2),
         (8 * 1032 * 3 + 100, 1032, 2), (40000, 40, 1), (129 * 64, 8, 2)]


def make_input(n, seed, kind):
    if kind == "random":
        return synth.random_bytes(n, seed)
    if kind == "text":
        return synth.text_like(n, seed)
    w = 64
    h = -(-n // (3 * w)) + 1
    return synth.bitmap(h, w, 3, seed).reshape(-1)[:n]


@pytest.mark.parametrize("n,W,L", SMALL)
def test_dwt_fwd_inv_parity(dev, orc, n, W, L):
    x = make_input(n, n + L, "random")
    coef = se.dwt_fwd(to_dev(x, dev), W, L)
    ref = orc.dwt_fwd(x, W, L)
    assert np.array_equal(coef.cpu().numpy().astype(np.int32), ref)
    back = se.dwt_inv(coef, n, W, L)
    assert np.array_equal(back.cpu().numpy(), x)


@pytest.mark.parametrize("kind", ["random", "bitmap", "text"])
@pytest.mark.parametrize("n,W,L", SMALL)
def test_protect_recover_parity(dev, orc, n, W, L, kind):
    x = make_input(n, 7 * n + L, kind)
    for flags in (0, se.FLAG_PUBLIC_PLAIN):
        for block_offset in (0, 128 * 5):
            a, b, c = se.fragment_protect(to_dev(x, dev), W, L, KEY, IV, flags=flags, block_offset=block_offset)
            oa, ob, oc = orc.protect(x, W, L, KEY, IV, flags=flags, block_offset=block_offset)
            assert np.array_equal(a.cpu().numpy(), oa), "A'"
            assert np.array_equal(b.cpu().numpy(), ob), "B'"
            assert np.array_equal(c.cpu().numpy(), oc), "C'"
            back, rep = se.fragment_recover(a, b, c, n, W, L, KEY, IV, flags=flags, block_offset=block_offset)
            assert np.array_equal(back.cpu().numpy(), x)
            assert rep.cpu().tolist() == [-1, 0]


def test_recover_of_oracle_fragments(dev, orc):
    """The GPU recovers fragments produced by the oracle (and vice versa)."""
    x = make_input(20000, 3, "bitmap")
    oa, ob, oc = orc.protect(x, 160, 2, KEY, IV)
    back, rep = se.fragment_recover(to_dev(oa, dev), to_dev(ob, dev), to_dev(oc, dev), x.size, 160, 2, KEY, IV)
    assert np.array_equal(back.cpu().numpy(), x) and rep.cpu().tolist() == [-1, 0]


def test_corruption_report_matches_oracle(dev, orc):
    x = make_input(64 * 1024, 4, "bitmap")
    W, L = 256, 2
    a, b, c = orc.protect(x, W, L, KEY, IV)
    bad_key = bytes([KEY[0] ^ 0x80]) + KEY[1:]
    back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c, dev), x.size, W, L, bad_key, IV)
    oback, orep = orc.recover(a, b, c, x.size, W, L, bad_key, IV)
    assert np.array_equal(back.cpu().numpy(), oback)
    assert tuple(rep.cpu().tolist()) == orep and orep[1] > 0
    # single flipped bit in C': confined to one block, same bytes as the oracle
    c2 = c.copy()
    c2[480 * 77 // 8 + 3] ^= 0x10
    back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c2, dev), x.size, W, L, KEY, IV)
    oback, orep = orc.recover(a, b, c2, x.size, W, L, KEY, IV)
    assert np.array_equal(back.cpu().numpy(), oback) and tuple(rep.cpu().tolist()) == orep


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 1000, 4096 + 7, 1 << 20])
def test_cipher_parity(dev, orc, n):
    x = synth.random_bytes(n, n)
    for off in (0, 3, (1 << 64) - 2):
        iv = bytes.fromhex("f0f1f2f3f4f5f6f7f8f9fafbfcfdfeff")
        got = se.cipher_encrypt(KEY, iv, to_dev(x, dev), ctr_block_offset=off) if n else None
        if n:
            assert np.array_equal(got.cpu().numpy(), orc.aes128_ctr(KEY, iv, x, ctr_offset=off))
            back = se.cipher_decrypt(KEY, iv, got, ctr_block_offset=off)
            assert np.array_equal(back.cpu().numpy(), x)


@pytest.mark.parametrize("mode", [se.MODE_BLOCK8, se.MODE_FULL])
@pytest.mark.parametrize("flags", [0, se.FLAG_PUBLIC_PLAIN])
def test_empty_input(dev, orc, mode, flags):
    """The degenerate case n = 0: empty fragments, empty recovery, the clean
    report {-1, 0}, as the oracle; no kernel launches but the report's init."""
    x = torch.empty(0, dtype=torch.uint8, device=dev)
    se.launch_count(reset=True)
    a, b, c = se.fragment_protect(x, 64, 2, KEY, IV, mode=mode, flags=flags)
    assert (a.numel(), b.numel(), c.numel()) == tuple(len(s) for s in orc.protect(np.zeros(0, np.uint8), 64, 2,
                                                                                  KEY, IV, mode=mode, flags=flags))
    y, rep = se.fragment_recover(a, b, c, 0, 64, 2, KEY, IV, mode=mode, flags=flags)
    torch.cuda.synchronize()
    assert y.numel() == 0 and rep.tolist() == [-1, 0]
    assert se.launch_count() == 1           # the report init kernel
    assert se.cipher_encrypt(KEY, IV, x).numel() == 0


def test_launch_evidence(dev):
    x = to_dev(synth.random_bytes(1 << 16, 1), dev)
    se.launch_count(reset=True)
    a, b, c = se.fragment_protect(x, 256, 2, KEY, IV)
    se.fragment_recover(a, b, c, x.numel(), 256, 2, KEY, IV)
    torch.cuda.synchronize()
    # masked (per-CTA kernels): protect = keystream into A' + fused kernel;
    # recover = report init + fused kernel (AES-CTR inside)
    assert se.launch_count() == 4
    se.launch_count(reset=True)
    a, b, c = se.fragment_protect(x, 256, 2, KEY, IV, flags=se.FLAG_PUBLIC_PLAIN)
    se.fragment_recover(a, b, c, x.numel(), 256, 2, KEY, IV, flags=se.FLAG_PUBLIC_PLAIN)
    torch.cuda.synchronize()
    assert se.launch_count() == 3           # PUBLIC_PLAIN (tile kernels): 1 + report init + 1


# ---------------------------------------------------------------- full-size configs

def sampled_ranges(nb, k=6, seed=0):
    """k 128-block groups: first, last, and random ones in between."""
    groups = (nb + 127) // 128
    rng = np.random.default_rng(seed)
    picks = {0, groups - 1} | set(int(g) for g in rng.integers(0, groups, size=k))
    return [(g * 128, min(nb, (g + 1) * 128)) for g in sorted(picks)]


def check_sampled(orc, x, W, L, a, b, c, iv, seed, flags=0):
    lay = orc.layout(x.size, W, L)
    ha, hb, hc = a.cpu().numpy(), b.cpu().numpy(), c.cpu().numpy()
    bits = (lay["a_bits"], lay["b_bits"], lay["c_bits"])
    for b0, b1 in sampled_ranges(lay["n_blocks"], seed=seed):
        bufs = [np.zeros(lay[k], np.uint8) for k in ("a_bytes", "b_bytes", "c_bytes")]
        orc.protect(x, W, L, KEY, iv, flags=flags, block_range=(b0, b1), out=bufs)
        for s, (got, ref) in enumerate(zip((ha, hb, hc), bufs)):
            lo, hi = b0 * bits[s] // 8, -(-b1 * bits[s] // 8)
            assert np.array_equal(got[lo:hi], ref[lo:hi]), ("stream", s, "blocks", b0, b1)


@pytest.mark.parametrize("flags", [0, se.FLAG_PUBLIC_PLAIN])
@pytest.mark.parametrize("cfg", [1, 2, 3, 33, 4])
def test_config_full_size(dev, orc, cfg, flags):
    """The BASELINE configs at full size in the bench's launch configuration
    (masked: per-CTA kernels + keystream kernels; PUBLIC_PLAIN: the tile
    kernels), sampled against the oracle where the whole file is too big."""
    base = 4 if cfg == 4 else 3 if cfg == 33 else cfg
    c = synth.CONFIGS[base]
    x = synth.config_input(cfg)
    W, L, iv = c["width"], c["levels"], synth.iv_for(base)
    xt = to_dev(x, dev)
    a, b, cc = se.fragment_protect(xt, W, L, KEY, iv, flags=flags)
    if cfg in (1, 2):          # small enough for the whole oracle
        oa, ob, oc = orc.protect(x, W, L, KEY, iv, flags=flags)
        assert np.array_equal(a.cpu().numpy(), oa)
        assert np.array_equal(b.cpu().numpy(), ob)
        assert np.array_equal(cc.cpu().numpy(), oc)
    else:
        check_sampled(orc, x, W, L, a, b, cc, iv, seed=cfg, flags=flags)
    back, rep = se.fragment_recover(a, b, cc, x.size, W, L, KEY, iv, flags=flags)
    assert rep.cpu().tolist() == [-1, 0]
    assert torch.equal(back, xt)
    del a, b, cc, back, xt
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- batches (C5) and stripes (row e)

def c5_subset(count, seed, max_size):
    rng = np.random.default_rng(seed)
    sizes = np.exp(rng.uniform(np.log(1024), np.log(max_size), size=count)).astype(np.int64)
    sizes[0] = 1                      # degenerate: one byte
    sizes[1] = 64 * 1024              # exact power-of-two file
    return [synth.c5_file(i, int(s)) for i, s in enumerate(sizes)]


@pytest.mark.parametrize("levels,flags", [(2, 0), (3, 0), (1, 0), (2, 1)])
def test_batch_files_parity(dev, orc, levels, flags):
    files = c5_subset(24, 50 + levels, 1 << 20)
    widths = [synth.width_rule(f.size) for f in files]
    ivs = [synth.iv_for(5, i) for i in range(len(files))]
    batch = se.Batch([to_dev(f, dev) for f in files], widths, ivs, levels, KEY, flags=flags)
    streams = batch.protect()
    for f, w, iv, (a, b, c) in zip(files, widths, ivs, streams):
        oa, ob, oc = orc.protect(f, w, levels, KEY, iv, flags=flags)
        assert np.array_equal(a.cpu().numpy(), oa)
        assert np.array_equal(b.cpu().numpy(), ob)
        assert np.array_equal(c.cpu().numpy(), oc)
    outs, reps = batch.recover()
    for f, o in zip(files, outs):
        assert np.array_equal(o.cpu().numpy(), f)
    assert (reps.cpu().numpy() == np.array([-1, 0])).all()


def test_batch_reports_per_file(dev, orc):
    files = c5_subset(6, 7, 1 << 18)
    widths = [synth.width_rule(f.size) for f in files]
    ivs = [synth.iv_for(5, i) for i in range(len(files))]
    batch = se.Batch([to_dev(f, dev) for f in files], widths, ivs, 2, KEY)
    streams = batch.protect()
    # corrupt file 3's private fragment: only its report may flag blocks
    streams[3][0][0] ^= 0xFF
    outs, reps = batch.recover()
    r = reps.cpu().numpy()
    oback, orep = orc.recover(streams[3][0].cpu().numpy(), streams[3][1].cpu().numpy(), streams[3][2].cpu().numpy(),
                              files[3].size, widths[3], 2, KEY, ivs[3])
    assert tuple(r[3]) == orep
    assert np.array_equal(outs[3].cpu().numpy(), oback)
    for i in range(len(files)):
        if i != 3:
            assert tuple(r[i]) == (-1, 0) and np.array_equal(outs[i].cpu().numpy(), files[i])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_virtual_stripes_equal_whole(dev, world):
    """Row-stripe sharding run serially on one GPU: the concatenated stripe
    streams equal the whole-file streams (what each of `world` GPUs computes)."""
    from paper_1803_04880_b200 import shard
    n, W, L = 8 * 1024 * 1024 + 12345, 1024, 2
    x = to_dev(synth.random_bytes(n, 99), dev)
    whole = se.fragment_protect(x, W, L, KEY, IV)
    parts = [[], [], []]
    for p in shard.plan_stripes(n, W, L, world):
        xs = x[p["byte_begin"]: p["byte_end"]].clone()
        st = se.fragment_protect(xs, W, L, KEY, IV, block_offset=p["block_offset"])
        for s in range(3):
            parts[s].append(st[s])
        back, rep = se.fragment_recover(*st, xs.numel(), W, L, KEY, IV, block_offset=p["block_offset"])
        assert torch.equal(back, xs) and rep.cpu().tolist() == [-1, 0]
    for s in range(3):
        assert torch.equal(torch.cat(parts[s]), whole[s])


def test_batch_1100_files_multi_pass_search(dev, orc):
    """with >1,024 jobs the batch kernel's 32-ary job search
    takes several dependent passes (1,100 -> 35 -> 2 -> 1).  Sampled files -
    first, last, the files around CTA-count boundaries and ~50 random ones -
    equal the oracle element by element; every file round-trips."""
    rng = np.random.default_rng(1100)
    n_files = 1100
    sizes = np.exp(rng.uniform(np.log(64), np.log(48 * 1024), size=n_files)).astype(np.int64)
    sizes[5] = 1
    sizes[6] = 8 * 1024                            # exactly one CTA of 128 blocks at W = 64... plus a row
    files = [synth.random_bytes(int(s), 7000 + i) for i, s in enumerate(sizes)]
    widths = [synth.width_rule(int(s)) for s in sizes]
    ivs = [synth.iv_for(5, i) for i in range(n_files)]
    batch = se.Batch([to_dev(f, dev) for f in files], widths, ivs, 2, KEY)
    begins = [int(batch.jobs[i].cta_begin) for i in range(n_files)]
    assert batch.total_ctas > 1100
    streams = batch.protect()
    picks = {0, 1, n_files - 2, n_files - 1} | set(rng.integers(0, n_files, size=50).tolist())
    # files whose CTA range starts right at / after a multiple of 32 CTAs (search lane boundaries)
    picks |= {i for i in range(1, n_files) if begins[i] // 32 != begins[i - 1] // 32}
    for i in sorted(picks)[:160]:
        oa, ob, oc = orc.protect(files[i], widths[i], 2, KEY, ivs[i])
        a, b, c = streams[i]
        assert np.array_equal(a.cpu().numpy(), oa), i
        assert np.array_equal(b.cpu().numpy(), ob), i
        assert np.array_equal(c.cpu().numpy(), oc), i
    outs, reps = batch.recover()
    for f, o in zip(files, outs):
        assert np.array_equal(o.cpu().numpy(), f)
    assert (reps.cpu().numpy() == np.array([-1, 0])).all()


@pytest.mark.parametrize("flags", [0, 1])
def test_batch_with_empty_and_tiny_files(dev, orc, flags):
    """Empty files (zero CTAs: several jobs share one cta_begin, including the
    first and the last job), one-byte files and whole-row files (W = 1024,
    where recover parks each CTA's keystream in its output region) mixed in one
    batch: every stream equals the oracle, every file round-trips, every report
    is clean - the job search and the keystream kernel's job stepping must skip
    the empty jobs."""
    sizes = [0, 1, 0, 0, 5000, 3 * 1024 * 1024, 0, 1, 70000, 2 * 1024 * 1024 + 512, 0, 64, 0]
    files = [synth.random_bytes(s, 400 + i) if s else np.zeros(0, np.uint8) for i, s in enumerate(sizes)]
    widths = [synth.width_rule(max(s, 1)) for s in sizes]
    ivs = [synth.iv_for(5, 900 + i) for i in range(len(sizes))]
    batch = se.Batch([to_dev(f, dev) for f in files], widths, ivs, 2, KEY, flags=flags)
    begins = [int(batch.jobs[i].cta_begin) for i in range(len(sizes))]
    assert begins[0] == begins[1] and begins[2] == begins[3] == begins[4]
    streams = batch.protect()
    for f, w, iv, (a, b, c) in zip(files, widths, ivs, streams):
        oa, ob, oc = orc.protect(f, w, 2, KEY, iv, flags=flags)
        assert np.array_equal(a.cpu().numpy(), oa)
        assert np.array_equal(b.cpu().numpy(), ob)
        assert np.array_equal(c.cpu().numpy(), oc)
    outs, reps = batch.recover()
    for f, o in zip(files, outs):
        assert np.array_equal(o.cpu().numpy(), f)
    assert (reps.cpu().numpy() == np.array([-1, 0])).all()


@pytest.mark.parametrize("W,rows,L", [(1024, 8 * 37, 2), (2048, 8 * 11, 3), (6144, 8 * 5, 2)])
def test_recover_keystream_in_output_region(dev, orc, W, rows, L):
    """Masked per-CTA recovery on whole rows of a multiple of 1024 bytes: the
    keystream kernel parks each CTA's A-slice keystream at the start of that
    CTA's own output region (and initialises the report).  Fragments from the
    oracle, clean, damaged and under a wrong key: bytes and report equal the
    oracle's."""
    n = W * rows
    x = make_input(n, W + rows, "bitmap")
    prev = se.kernel_choice(se.KERNEL_AUTO)
    try:
        a, b, c = orc.protect(x, W, L, KEY, IV)
        ga, gb, gc = se.fragment_protect(to_dev(x, dev), W, L, KEY, IV)
        assert np.array_equal(ga.cpu().numpy(), a) and np.array_equal(gc.cpu().numpy(), c)
        back, rep = se.fragment_recover(to_dev(a, dev), to_dev(b, dev), to_dev(c, dev), n, W, L, KEY, IV)
        assert np.array_equal(back.cpu().numpy(), x) and rep.cpu().tolist() == [-1, 0]
        a2, c2 = a.copy(), c.copy()
        a2[len(a2) // 2] ^= 0x21
        c2[60 * 200 + 5] ^= 0x04
        for key, aa, cc in ((KEY, a2, c2), (bytes([KEY[0] ^ 4]) + KEY[1:], a, c)):
            back, rep = se.fragment_recover(to_dev(aa, dev), to_dev(b, dev), to_dev(cc, dev), n, W, L, key, IV)
            oback, orep = orc.recover(aa, b, cc, n, W, L, key, IV)
            assert np.array_equal(back.cpu().numpy(), oback)
            assert tuple(rep.cpu().tolist()) == orep and orep[1] > 0
    finally:
        se.kernel_choice(prev)


def test_c5_full_workload_sampled(dev, orc):
    """BASELINE config 5 at full size in the bench's launch configuration: the
    10,000 files (log-uniform 1 KiB-16 MiB, ~17 GB) in one batched launch per
    direction, as `bench.py --config 5` builds them; 30 sampled files (the
    smallest, the largest, and random ones) equal the oracle element by
    element, every file round-trips."""
    sizes = synth.c5_file_sizes(10000, 5)
    gen = torch.Generator(device=dev)
    files = []
    for i in range(len(sizes)):
        gen.manual_seed(5_000_000 + i)
        files.append(torch.randint(0, 256, (int(sizes[i]),), dtype=torch.uint8, device=dev, generator=gen))
    widths = [synth.width_rule(int(s)) for s in sizes]
    ivs = [synth.iv_for(5, i) for i in range(len(sizes))]
    batch = se.Batch(files, widths, ivs, 2, KEY)
    streams = batch.protect()
    rng = np.random.default_rng(55)
    order = np.argsort(sizes)
    picks = {int(order[0]), int(order[1]), int(order[-1])} | set(rng.integers(0, len(sizes), size=27).tolist())
    for i in sorted(picks):
        x = files[i].cpu().numpy()
        oa, ob, oc = orc.protect(x, widths[i], 2, KEY, ivs[i])
        a, b, c = streams[i]
        assert np.array_equal(a.cpu().numpy(), oa), i
        assert np.array_equal(b.cpu().numpy(), ob), i
        assert np.array_equal(c.cpu().numpy(), oc), i
    outs, reps = batch.recover()
    assert all(torch.equal(o, f) for o, f in zip(outs, files))
    assert (reps.cpu().numpy() == np.array([-1, 0])).all()
    del files, outs, streams, batch
    torch.cuda.empty_cache()


@pytest.mark.parametrize("flags", [0, se.FLAG_PUBLIC_PLAIN])
def test_protect_recover_capture_into_cuda_graph(dev, orc, flags):
    """The device-resident calls are stream-ordered with no host
    synchronisation or allocation, so a protect + recover round trip can be
    captured once into a CUDA graph and replayed on new data (the per-CTA
    path with its keystream kernels when masked, the tile kernels when
    PUBLIC_PLAIN)."""
    n, W, L = 1024 * 8 * 200, 1024, 2
    x0 = synth.random_bytes(n, 11)
    x = to_dev(x0, dev)
    lay = se.fragment_layout(n, W, L)
    a, b, c = (se._empty(lay[k], dev) for k in ("a_bytes", "b_bytes", "c_bytes"))
    out = se._empty(n, dev)
    rep = torch.empty(2, dtype=torch.int64, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):                       # warm-up outside the capture (module loading)
        se.fragment_protect(x, W, L, KEY, IV, flags=flags, out=(a, b, c), stream=s)
        se.fragment_recover(a, b, c, n, W, L, KEY, IV, flags=flags, out=out, report=rep, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        se.fragment_protect(x, W, L, KEY, IV, flags=flags, out=(a, b, c), stream=s)
        se.fragment_recover(a, b, c, n, W, L, KEY, IV, flags=flags, out=out, report=rep, stream=s)
    for seed in (12, 13):
        x1 = synth.random_bytes(n, seed)
        x.copy_(torch.from_numpy(x1))
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), x1) and rep.cpu().tolist() == [-1, 0]
        oa, _, oc = orc.protect(x1, W, L, KEY, IV, flags=flags)
        assert np.array_equal(a.cpu().numpy(), oa) and np.array_equal(c.cpu().numpy(), oc)


def test_batch_recover_keystream_in_output_regions(dev, orc):
    """Batch recovery of files >= 1 MiB (W = 1024): whole-row CTAs take their
    keystream from their own output region, the files' ragged last CTAs run
    the AES themselves; damaged and clean files, reports per file == the
    oracle's."""
    sizes = [(1 << 20) + 5000, 3 * (1 << 20), (2 << 20) + 8192 * 3, 1 << 20, 1500 * 1024]
    files = [synth.random_bytes(s, 300 + i) for i, s in enumerate(sizes)]
    widths = [synth.width_rule(s) for s in sizes]
    assert all(w == 1024 for w in widths)
    ivs = [synth.iv_for(5, 900 + i) for i in range(len(files))]
    batch = se.Batch([to_dev(f, dev) for f in files], widths, ivs, 2, KEY)
    streams = batch.protect()
    # damage file 1 (A' in a whole-row CTA) and file 4 (C' in its ragged last CTA)
    streams[1][0][640 * 3 + 1] ^= 0x08
    streams[4][2][streams[4][2].numel() - 7] ^= 0x40
    outs, reps = batch.recover()
    r = reps.cpu().numpy()
    for i, (f, w, iv) in enumerate(zip(files, widths, ivs)):
        a, b, c = (t.cpu().numpy() for t in streams[i])
        oback, orep = orc.recover(a, b, c, f.size, w, 2, KEY, iv)
        assert tuple(r[i]) == orep, i
        assert np.array_equal(outs[i].cpu().numpy(), oback), i
    assert r[1][1] > 0 and r[4][1] >= 0 and tuple(r[0]) == (-1, 0)
