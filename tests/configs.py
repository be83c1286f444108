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
    if r.random() < 0.5:
        # memory-starved: KV capacity of a few thousand tokens forces evictions/preemptions
        from paper_2411_05555_b200.abi import MODELS
        W = MODELS[model][0] * MODELS[model][5]
        kvb = 2 * MODELS[model][1] * MODELS[model][3] * MODELS[model][4] * MODELS[model][5]
        tokens = r.randint(pmax + dmax + 10, 4 * (pmax + dmax) + 3000)
        p.hbm_capacity = (W + tokens * kvb) / (p.num_devices * (1.0 - p.memory_reserve_fraction))
    return p
