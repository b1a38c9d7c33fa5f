"""Does schedule()'s API latency change after the bench's other secondary
measurements?  (bench reported 46 ms; alone it is ~1.2 ms.)"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import bench

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
print("fresh", bench.api_latency_measure(dev)["ms_per_call"], flush=True)
for name, fn in (("mode_a_c1", lambda: bench.mode_a_measure(dev, "c1")), ("mode_a_c2", lambda: bench.mode_a_measure(dev, "c2")),
                 ("dp_c1_grid", lambda: bench.dp_measure(dev)), ("schedule_c4", lambda: bench.c4_measure(dev)),
                 ("random_c5", lambda: bench.random_measure(dev, "c5")), ("random_c3", lambda: bench.random_measure(dev, "c3")),
                 ("dp_c4b", lambda: bench.dp_c4b_measure(dev))):
    t0 = time.perf_counter()
    fn()
    print(name, "took", time.perf_counter() - t0, "then api ms", bench.api_latency_measure(dev)["ms_per_call"], flush=True)
torch.cuda.empty_cache()
print("after empty_cache", bench.api_latency_measure(dev)["ms_per_call"])
print("mem", torch.cuda.memory_reserved() / 1e9, "GB reserved")
