"""Cross-rank aggregation of bench results (one process per GPU, weak scaling).

Requests are independent (north_star: no collective on the data path), so the
only cross-rank traffic is this end-of-run reduction: SLO-satisfying and total
requests are summed over ranks, device time and wall time take the max over
ranks, and value = summed requests / max time."""


def aggregate(dist, sat, tot, dev_s, wall_s):
    if dist is None:
        return sat, tot, dev_s, wall_s
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    s = torch.tensor([float(sat), float(tot)], dtype=torch.float64, device=dev)
    m = torch.tensor([float(dev_s), float(wall_s)], dtype=torch.float64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return s[0].item(), s[1].item(), m[0].item(), m[1].item()
