"""Point generators shared by the CPU (emulator) and GPU parity tests.

BASELINE.json configs 1-3 (at parity sizes) and the SPEC.md:469 randomized
small-config generator (<= 4 instances, <= 50 requests), extended with
memory-starved instances so eviction and preemption paths are exercised."""
from __future__ import annotations

import random

from paper_2411_05555_b200.abi import make_point

POLICIES = ["unified", "splitwise", "accellm"]


def closed_form_point():
    # one request 512/10 on one H100 pair, eff (0.5,1,1)
    return make_point(model="llama2-70b", device="h100", policy="accellm", instances=2, num_requests=1,
                      prompt=512, decode=10, arrival="fixed", rate=1.0, eff=(0.5, 1.0, 1.0))


def config1(seed=0, n=1000):
    # BASELINE config 1: Llama-2 7B, 4 H100 instances (2 AcceLLM pairs), Poisson 2/s, fixed 512/10
    return make_point(model="llama2-7b", device="h100", policy="accellm", instances=4, num_requests=n,
                      rate=2.0, prompt=512, decode=10, seed=seed)


def config2(policy, rate, seed=0, n=10000):
    # BASELINE config 2: Llama-2 70B, 8 H100, conversation-shaped (builder preset)
    return make_point(model="llama2-70b", device="h100", policy=policy, instances=8, num_requests=n,
                      rate=rate, workload="conversation", seed=seed)


def config3(policy, rate, seed=0, n=10000):
    # BASELINE config 3: Llama-2 70B on 910B2, 8 instances, coding-shaped (builder preset)
    return make_point(model="llama2-70b", device="910b2", policy=policy, instances=8, num_requests=n,
                      rate=rate, workload="coding", seed=seed)


def random_small(i: int, max_req: int = 50):
    r = random.Random(1000 + i)
    policy = POLICIES[i % 3]
    inst = r.choice([2, 4]) if policy != "splitwise" else r.choice([2, 3, 4])
    model = r.choice(["llama2-7b", "llama2-70b"])
    device = r.choice(["h100", "910b2"])
    pmin = r.randint(1, 400)
    pmax = pmin + r.randint(0, 600)
    dmin = r.randint(1, 100)
    dmax = dmin + r.randint(0, 300)
    rate = r.choice([0.5, 2.0, 8.0, 30.0, 200.0])
    p = make_point(model=model, device=device, policy=policy, instances=inst, num_requests=r.randint(1, max_req),
                   rate=rate, workload=(pmin, pmax, dmin, dmax), seed=r.randint(0, 1 << 30),
                   arrival=r.choice(["poisson", "poisson", "fixed"]), link=r.choice(["striped", "single"]),
                   prefill_budget=r.choice([8192, 2048, 700]),
                   warmup_s=r.choice([0.0, 0.0, 1.0]))
    if policy == "splitwise" and r.random() < 0.4:
        p.splitwise_cobatch = 1  # high-load co-batching
    if (i * 7919) % 5 == 0:
        p.first_token_decode = 1  # first token from the first decode step (SPEC.md:273 alternative)
    if r.random() < 0.5:
        # memory-starved: KV capacity of a few thousand tokens forces evictions/preemptions
        from paper_2411_05555_b200.abi import MODELS
        W = MODELS[model][0] * MODELS[model][5]
        kvb = 2 * MODELS[model][1] * MODELS[model][3] * MODELS[model][4] * MODELS[model][5]
        tokens = r.randint(pmax + dmax + 10, 4 * (pmax + dmax) + 3000)
        p.hbm_capacity = (W + tokens * kvb) / (p.num_devices * (1.0 - p.memory_reserve_fraction))
    return p


def random_ext(i: int, max_req: int = 200):
    """AcceLLM with the timer-driven extensions (docs/SEMANTICS.md §6b):
    degraded mode and/or inter-pair leveling, short timer periods so small
    runs see many ticks, memory-starved instances so degraded mode triggers."""
    r = random.Random(5000 + i)
    inst = r.choice([4, 4, 6, 8])
    model = r.choice(["llama2-7b", "llama2-70b"])
    device = r.choice(["h100", "910b2"])
    pmin = r.randint(1, 300)
    pmax = pmin + r.randint(0, 500)
    dmin = r.randint(1, 60)
    dmax = dmin + r.randint(0, 200)
    flags = r.choice([(True, False), (False, True), (True, True)])
    p = make_point(model=model, device=device, policy="accellm", instances=inst, num_requests=r.randint(20, max_req),
                   rate=r.choice([4.0, 16.0, 60.0, 200.0]), workload=(pmin, pmax, dmin, dmax),
                   seed=r.randint(0, 1 << 30), arrival=r.choice(["poisson", "poisson", "fixed"]),
                   link=r.choice(["striped", "single"]), prefill_budget=r.choice([8192, 2048, 700]),
                   degraded=flags[0], leveling=flags[1], timer_s=r.choice([0.01, 0.05, 0.2, 1.0]),
                   trigger_ticks=r.choice([0, 1, 2]), leveling_fraction=r.choice([0.0, 0.5, 5.0]),
                   degraded_redundancy=r.choice([0.0, 0.9]), degraded_exit_fill=r.choice([0.0, 0.3, 0.9]),
                   dual_copy_fraction=r.choice([0.0, 0.5]))
    if (i * 7919) % 4 == 1:
        p.first_token_decode = 1
    if r.random() < 0.6:
        from paper_2411_05555_b200.abi import MODELS
        W = MODELS[model][0] * MODELS[model][5]
        kvb = 2 * MODELS[model][1] * MODELS[model][3] * MODELS[model][4] * MODELS[model][5]
        tokens = r.randint(pmax + dmax + 10, 6 * (pmax + dmax) + 4000)
        p.hbm_capacity = (W + tokens * kvb) / (p.num_devices * (1.0 - p.memory_reserve_fraction))
    return p


def ext_long_points(n: int = 800):
    """Longer extension runs: many degraded entries/exits, heavy leveling."""
    return [
        make_point(policy="accellm", instances=4, rate=12.0, num_requests=n, workload="heavy", reserve=0.5, seed=3,
                   degraded=True, timer_s=0.2),
        make_point(policy="accellm", instances=8, rate=30.0, num_requests=n, workload="heavy", reserve=0.5, seed=4,
                   degraded=True, leveling=True, timer_s=0.1, trigger_ticks=1),
        make_point(policy="accellm", instances=6, rate=10.0, num_requests=n, workload="mixed", seed=5,
                   leveling=True, timer_s=0.05, leveling_fraction=2.0),
        make_point(policy="accellm", instances=16, rate=40.0, num_requests=n, workload="mixed", seed=6,
                   leveling=True, degraded=True, device="910b2", reserve=0.4, timer_s=0.1),
    ]
