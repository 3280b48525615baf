"""Random valid plans for property tests (random DP <= 4, per-pipeline PP <= 2,
random member counts, whole-head / 16-column splits, random m_i summing to B/b, random standby)."""
import numpy as np

from paper_2410_13333_b200.plans import stage, plan, pipe


def _rand_split(rng, total, k, gran):
    units = total // gran
    cuts = sorted(rng.choice(np.arange(1, units), size=k - 1, replace=False)) if k > 1 else []
    b = [0] + list(cuts) + [units]
    return [(b[i + 1] - b[i]) * gran for i in range(k)]


def random_plan(rng, cfg, world_max=8, B=8, b=2, max_dp=4, max_pp=2):
    ranks = list(rng.permutation(world_max))
    dp = int(rng.integers(1, min(max_dp, world_max) + 1))
    pipes = []
    used = 0
    for i in range(dp):
        pp = int(rng.integers(1, max(1, min(max_pp, cfg.n_layers, world_max - used - (dp - i - 1))) + 1))
        bounds = [0] + sorted(rng.choice(np.arange(1, cfg.n_layers), size=pp - 1, replace=False).tolist()) + [cfg.n_layers] if pp > 1 else [0, cfg.n_layers]
        stages = []
        for j in range(pp):
            left = world_max - used - (dp - i - 1) - (pp - j - 1)
            kmax = max(1, min(cfg.n_heads, left, 4, cfg.ffn // 16, cfg.vocab // 16))
            k = int(rng.integers(1, kmax + 1))
            rr = ranks[used:used + k]
            used += k
            stages.append(stage(rr, _rand_split(rng, cfg.n_heads, k, 1), _rand_split(rng, cfg.ffn, k, 16),
                                _rand_split(rng, cfg.vocab, k, 16), [bounds[j], bounds[j + 1]]))
        pipes.append(stages)
    total_m = B // b
    cuts = sorted(rng.integers(0, total_m + 1, size=dp - 1).tolist())
    ms = [c1 - c0 for c0, c1 in zip([0] + cuts, cuts + [total_m])]
    n_standby = int(rng.integers(0, world_max - used + 1))
    world = used + n_standby
    standby = ranks[used:world]
    p = plan([pipe(st, m) for st, m in zip(pipes, ms)], b, B, standby=standby)
    # renumber ranks densely into [0, world)
    rank_map = {r: i for i, r in enumerate(sorted([r for pp in p["pipes"] for st in pp["stages"] for r in st["ranks"]] + standby))}
    for pp in p["pipes"]:
        for st in pp["stages"]:
            st["ranks"] = [rank_map[r] for r in st["ranks"]]
    p["standby"] = [rank_map[r] for r in standby]
    return p, world
