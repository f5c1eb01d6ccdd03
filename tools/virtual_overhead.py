"""Orchestration overhead of a k-shard context, measured on ONE GPU: the same
job run as 1 shard (an NCCL context) and as k virtual shards (one DevCtx +
worker thread per shard, all on this GPU, host-gathered records).  The total
work is the same, so the difference is what sharding itself costs (not a
scaling measurement: the shards share one GPU)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_17746_b200 as ws  # noqa: E402
from bench import splitmix_starts  # noqa: E402

jobs = {
    "c3": lambda s: s.count_range(0, 10**12 + 1),
    "c1": lambda s: s.count_range(0, 10**9 + 1),
    "c5": lambda s: s.count_intervals(splitmix_starts(42, 4096, 2**32, 2**44), 2**24),
}
out = {}
for k in (1, 2, 8):
    if k > 1:
        os.environ["WHEELSIEVE_VIRTUAL_SHARDS"] = "1"
        os.environ["WHEELSIEVE_BUCKET_BUDGET"] = str(1 << 30)
    s = ws.Sieve(devices=[0] * k)
    for name, f in jobs.items():
        f(s)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            f(s)
            ts.append((time.perf_counter() - t0) * 1e3)
        out.setdefault(name, {})[f"{k} shard{'s' if k > 1 else ''}"] = round(float(np.median(ts)), 3)
    s.close()
print(json.dumps({"what": "median wall ms per call on one B200 (k virtual shards share it)",
                  "results": out}))
