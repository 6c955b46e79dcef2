"""gpu-let executor on a B200: green-context confinement (%smid audit), the
SM counts of the partition grid, co-resident gpu-lets, submit/poll ordering,
and the C-ABI error paths (SURVEY §4.4 integration layer)."""
import numpy as np
import pytest

import synthgen
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c():
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    ctx.mid = ctx.load_model(0, "lenet5", synthgen.weight_file("lenet5"))
    yield ctx
    ctx.close()


@pytest.mark.parametrize("p,q", [(20, 80), (40, 60), (50, 50), (60, 40), (80, 20)])
def test_pair_confinement(c, p, q):
    (a, na), (b, nb) = c.create_gpulets(0, [p, q])
    try:
        # SM-pair split (no co-scheduling groups): a p % gpu-let holds p % of the
        # 148 SMs rounded to an even count, so (p, 100 - p) pairs split exactly
        share = {20: 30, 40: 60, 50: 74, 60: 88, 80: 118}
        assert (na, nb) == (share[p], share[q]) and na + nb == 148
        sa, sb = c.gpulet_smids(a), c.gpulet_smids(b)
        assert len(set(sa)) == na and len(set(sb)) == nb      # one CTA per SM
        assert not set(sa) & set(sb)                          # disjoint SM sets
    finally:
        c.destroy_gpulet(a)
        c.destroy_gpulet(b)


def test_partition_errors(c):
    from paper_2109_01611_b200 import gpulet
    with pytest.raises(gpulet.GpuletError) as e:
        c.create_gpulet(0, 30)
    assert e.value.code == -2
    a, _ = c.create_gpulet(0, 60)
    try:
        with pytest.raises(gpulet.GpuletError) as e:
            c.create_gpulet(0, 60)
        assert e.value.code == -4
    finally:
        c.destroy_gpulet(a)


def test_submit_poll_fifo_and_errors(c):
    import torch
    from paper_2109_01611_b200 import gpulet
    g, _ = c.create_gpulet(0, 100)
    try:
        x = to_dev_bf16(synthgen.mnist_batch(32))
        y = torch.empty(320, device="cuda")
        tickets = [c.submit_batch(g, c.mid, x, y, 32, 5.0) for _ in range(100)]
        got = []
        while len(got) < 100:
            got += [r.ticket for r in c.poll()]
        assert got == tickets                                  # FIFO per gpu-let
        with pytest.raises(gpulet.GpuletError) as e:
            c.submit_batch(g, c.mid, x, y, 33)
        assert e.value.code == -3
        with pytest.raises(gpulet.GpuletError) as e:
            c.submit_batch(g, 99, x, y, 1)
        assert e.value.code == -6
    finally:
        c.destroy_gpulet(g)
    with pytest.raises(gpulet.GpuletError) as e:
        c.submit_batch(g, c.mid, x, y, 1)
    assert e.value.code == -5


def test_corun_overlap(c):
    """Two gpu-lets execute concurrently: their device busy intervals overlap."""
    import torch
    (a, _), (b, _) = c.create_gpulets(0, [50, 50])
    try:
        x = to_dev_bf16(synthgen.mnist_batch(32))
        ya, yb = torch.empty(320, device="cuda"), torch.empty(320, device="cuda")
        for _ in range(200):
            c.submit_batch(a, c.mid, x, ya, 32)
            c.submit_batch(b, c.mid, x, yb, 32)
        recs = []
        while len(recs) < 400:
            recs += c.poll()
        ia = [(r.t_start_ns, r.t_end_ns) for r in recs if r.gpulet == a]
        ib = [(r.t_start_ns, r.t_end_ns) for r in recs if r.gpulet == b]
        assert max(ia)[0] > min(ib)[0] and max(ib)[0] > min(ia)[0]
        assert np.allclose(ya.cpu().numpy(), yb.cpu().numpy())
    finally:
        c.destroy_gpulet(a)
        c.destroy_gpulet(b)


def test_unconfined_pair_serves_and_places_one_cta_per_sm(c):
    """F4 "MPS(default)" analogue (gl_create_gpulets_unconfined): two executors on the
    primary context, CTA counts of the 20:80 split, placed by the hardware; each CTA
    holds a whole SM, so the two CTA sets land on distinct SMs; both serve batches
    that match the oracle."""
    import torch
    from oracle import models as omodels
    (a, na), (b, nb) = c.create_gpulets(0, [20, 80], unconfined=True)
    try:
        assert (na, nb) == (30, 118)
        sa, sb = c.gpulet_smids(a), c.gpulet_smids(b)
        assert len(set(sa)) == na and len(set(sb)) == nb and not set(sa) & set(sb)
        x = synthgen.model_input("lenet5", 8)
        for gid in (a, b):
            y = torch.empty(c.model_io(c.mid, 8)[1] // 4, device="cuda")
            c.wait(c.submit_batch(gid, c.mid, to_dev_bf16(x), y, 8, 10.0))
            ref = omodels.forward("lenet5", synthgen.weights("lenet5"), x)["logits"]
            got = y.cpu().numpy().astype(np.float64).reshape(ref.shape)
            assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max()
    finally:
        c.destroy_gpulet(a)
        c.destroy_gpulet(b)


@pytest.mark.parametrize("pcts", [[20, 20, 20], [20, 20, 20, 20], [20, 40, 20]])
def test_three_and_four_gpulets_per_gpu(c, pcts):
    """F4's "more than 2 gpu-lets per GPU": 3-4 green-context gpu-lets at their exact
    shares on disjoint SM sets, each serving LeNet-5 batches that match the oracle;
    a partition whose exact shares exceed 148 SMs is refused."""
    import torch
    from oracle import models as omodels
    from paper_2109_01611_b200 import gpulet
    share = {20: 30, 40: 60}
    x = synthgen.model_input("lenet5", 8)
    xd = to_dev_bf16(x)
    ys = [torch.empty(c.model_io(c.mid, 8)[1] // 4, device="cuda") for _ in pcts]
    torch.cuda.synchronize()
    made = c.create_gpulets(0, pcts)
    try:
        assert [n for _g, n in made] == [share[p] for p in pcts]
        seen = set()
        for gid, n in made:
            sm = set(c.gpulet_smids(gid))
            assert len(sm) == n and not (sm & seen)
            seen |= sm
        ref = omodels.forward("lenet5", synthgen.weights("lenet5"), x)["logits"]
        tickets = [c.submit_batch(gid, c.mid, xd, y, 8, 10.0) for (gid, _n), y in zip(made, ys)]
        for t, y in zip(tickets, ys):
            c.wait(t)
            got = y.cpu().numpy().astype(np.float64).reshape(ref.shape)
            assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max()
    finally:
        for gid, _n in made:
            c.destroy_gpulet(gid)
    with pytest.raises(gpulet.GpuletError):
        c.create_gpulets(0, [20, 20, 20, 40])
    (a, na), (b, nb) = c.create_gpulets(0, [50, 50])   # back to the two-slot layout
    try:
        assert (na, nb) == (74, 74) and not set(c.gpulet_smids(a)) & set(c.gpulet_smids(b))
    finally:
        c.destroy_gpulet(a)
        c.destroy_gpulet(b)
