"""Host-side logic of the slab-partitioned solve, on CPU:
the partition rule exported by libhmg (hmg_slab_partition) and the
torch.distributed bootstrap of bench.py / dist.py, exercised by a
world-size-2 gloo process group."""
import os
import socket

import numpy as np
import pytest


def test_partition_rule_tiles_every_level():
    from paper_2511_16808_b200 import hmg
    for n0, L, P in ((4097, 9, 8), (129, 4, 3), (385, 7, 8), (257, 6, 2), (641, 7, 4)):
        lo, hi, dist = hmg.slab_partition(n0, L, P)
        N = n0
        for l in range(L):
            assert lo[l, 0] == 0 and hi[l, -1] == N
            assert np.all(lo[l, 1:] == hi[l, :-1])
            if l > 0:   # coarse node I belongs to the rank owning fine node 2I
                for r in range(P):
                    if lo[l, r] < hi[l, r]:
                        for I in (lo[l, r], hi[l, r] - 1):
                            assert lo[l - 1, r] <= 2 * I < hi[l - 1, r]
            if dist[l]:   # distributed levels: every slab at least 2 G rows
                assert np.all(hi[l] - lo[l] >= 8)
            N = (N - 1) // 2 + 1
        assert dist[-1] == 0
        assert np.all(np.diff(dist) <= 0), "distributed levels must be a prefix"


def test_single_rank_partition_is_replicated():
    from paper_2511_16808_b200 import hmg
    lo, hi, dist = hmg.slab_partition(129, 4, 1)
    assert not dist.any() and hi[0, 0] == 129


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_16808_b200 import dist as hd
        uid = hd.share_unique_id(lambda: bytes(range(128)))
        t = hd.max_over_ranks(1.0 + rank)
        rows = hd.slab_rows(4097, 9, world, rank)
        q.put((rank, uid == bytes(range(128)), t, rows))
    finally:
        dist.destroy_process_group()


def test_gloo_bootstrap_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o[1] for o in out), "unique id not broadcast"
    assert all(o[2] == 2.0 for o in out), "max over ranks"
    assert out[0][3] == (0, 2048) and out[1][3] == (2048, 4097)


def test_setup_plan_config4_fits_8_ranks():
    """Partitioned build: BASELINE configs[4] at full size (768^2 x 384 cells,
    7 levels, element Vanka, c64).  On one GPU the modelled build peak is far above 180 GB;
    slab-partitioned over 8 ranks every rank's peak and its resident + FGMRES(20) bytes fit
    in 180 GB.  The kept rows of every partitioned level tile the level exactly, and each
    setup window holds its kept rows and G = 4 ghost rows (host-only: no device)."""
    from paper_2511_16808_b200 import hmg
    o = hmg.Options(dim=3, cells=(768, 768, 384), h=25.0, levels=7, smoother="element",
                    damping=[1.1, 0.7, 0.45, 0.6], dtype="c64")
    one = hmg.setup_plan(o, 1, 0)
    assert one["partitioned_levels"] == 0 and one["setup_peak_bytes"] > 180e9
    plans = [hmg.setup_plan(o, 8, r) for r in range(8)]
    nd = plans[0]["partitioned_levels"]
    assert nd >= 2
    for pl in plans:
        assert pl["setup_peak_bytes"] < 180e9
        assert pl["resident_bytes"] + pl["fgmres20_bytes"] < 180e9
    for l in range(nd):
        kept = sorted(pl["kept"][l] for pl in plans)
        assert kept[0][0] == 0 and all(a[1] == b[0] for a, b in zip(kept, kept[1:]))
        for pl in plans:
            (wl, wh), (kl, kh) = pl["window"][l], pl["kept"][l]
            assert wl <= max(0, kl - 4) and wh >= kh + 4 or wh == [385, 193, 97][l]
    # peak per rank scales down with the rank count (about 1/N of the level-0 work plus margins)
    assert max(p["setup_peak_bytes"] for p in plans) < 0.35 * one["setup_peak_bytes"]
