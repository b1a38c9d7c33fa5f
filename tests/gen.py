"""Instance generators used by the parity tests.

`random_stages` / `uniform_fleet` reproduce the reference's own test
generators (pkg/tests/test_scheduling.py:20-37) call for call, so with the
same numpy seeds they yield the very instances the reference's tests use —
built here from the engine's mirror types, which needs no reference package
on the GPU box.  `big_instance` makes larger DAG/chain instances with pairwise
links that take the proportional + hill-climb path.
"""

import numpy as np

from paper_2309_01172_b200 import refapi as M


def uniform_fleet(speeds, link=M.ZERO_LINK, gpu_gb=64.0, backups=()):
    peers = {str(i + 1): M.Peer(str(i + 1), peak_flops=s, gpu_bytes=gpu_gb * 2**30)
             for i, s in enumerate(speeds)}
    return M.Fleet(peers=peers, default_link=link, backup_pool=tuple(backups))


def random_stages(rng, n):
    stages = []
    for i in range(n):
        edges = ()
        if i > 0:
            src = int(rng.integers(0, i))
            edges = ((src, int(rng.integers(256, 65536))),)
        stages.append(M.Stage(index=i, label=f"s{i}", flops=float(rng.integers(10**5, 10**8)),
                              gpu_bytes=float(rng.integers(2**10, 2**24)),
                              cpu_bytes=1024.0, disk_bytes=512.0, in_edges=edges))
    return stages


def criterion6_instances(seed=2024, count=200):
    """Acceptance criterion 6 generator (pkg/tests/test_acceptance.py:141-156)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(2, 13))
        p = int(rng.integers(2, 5))
        stages = random_stages(rng, n)
        link = M.Link(float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7)))
        cap_gb = float(rng.uniform(0.7, 1.6)) * sum(s.gpu_bytes for s in stages) / 2**30
        fleet = uniform_fleet(list(rng.uniform(1e8, 1e9, p)), link=link, gpu_gb=cap_gb)
        out.append((stages, fleet))
    return out


def big_instance(rng, n, p, *, dag=True, frac=False, links=False, pressure=(0.05, 0.6)):
    st = []
    for i in range(n):
        edges = ()
        if i > 0:
            if dag:
                k = int(rng.integers(1, 3))
                srcs = sorted(set(int(x) for x in rng.integers(max(0, i - 4), i, k)))
            else:
                srcs = [i - 1]
            edges = tuple((s, int(rng.integers(256, 2**22))) for s in srcs)
        fl = float(rng.integers(10**9, 10**12)) + (float(rng.random()) if frac else 0.0)
        st.append(M.Stage(i, f"s{i}", fl, float(rng.integers(2**20, 2**30)),
                          float(rng.integers(1024, 2**20)), 512.0, edges))
    total = sum(s.gpu_bytes for s in st)
    peers = {str(k + 1): M.Peer(str(k + 1), peak_flops=float(rng.choice([59.5e12, 97.5e12, 82.58e12, 155.92e12])),
                                lam=float(rng.uniform(0.3, 1)), gpu_bytes=float(rng.uniform(*pressure)) * total)
             for k in range(p)}
    lk = {}
    if links:
        ids = list(peers)
        for _ in range(3 * p):
            a, b = rng.choice(ids, 2, replace=False)
            lk[(str(a), str(b))] = M.Link(float(rng.uniform(0, 0.02)), 8 / (float(rng.uniform(0.1, 100)) * 1e9))
    fleet = M.Fleet(peers=peers, default_link=M.Link(float(rng.uniform(0, 0.01)), 8 / (float(rng.uniform(0.1, 10)) * 1e9)),
                    links=lk, msg_ratio=float(rng.choice([1.0, 0.5, 0.3])))
    return st, fleet
