"""Probe: do two half-batches (B = 16 each) on two streams beat one B = 32 batch (c2)?
python tools/concurrency_probe.py"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_06363_b200 as rbs  # noqa: E402
from synth import CONFIGS, query_set, train_set  # noqa: E402

c = CONFIGS["c2"]
s0 = rbs.Solver(c.dim, c.m, c.blocks)
gr = s0.build_greedy(train_set(c), c.n)
W, A, f = gr["W"].contiguous(), gr["ANq"], gr["fn"]
s1 = rbs.Solver(c.dim, c.m, c.blocks).load_basis(W, A, f)
s2 = rbs.Solver(c.dim, c.m, c.blocks).load_basis(W, A, f)
mus = query_set(c)[:64]
st1, st2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


one = timeit(lambda: s0.solve_batch(mus[:32], want_a_n=False))
seq = timeit(lambda: (s1.solve_batch(mus[:16], want_a_n=False, stream=st1),
                      s2.solve_batch(mus[16:32], want_a_n=False, stream=st2)))


def par():
    th = [threading.Thread(target=lambda: s1.solve_batch(mus[:16], want_a_n=False, stream=st1)),
          threading.Thread(target=lambda: s2.solve_batch(mus[16:32], want_a_n=False, stream=st2))]
    for t in th:
        t.start()
    for t in th:
        t.join()


conc = timeit(par)


def par32():
    th = [threading.Thread(target=lambda: s1.solve_batch(mus[:32], want_a_n=False, stream=st1)),
          threading.Thread(target=lambda: s2.solve_batch(mus[32:64], want_a_n=False, stream=st2))]
    for t in th:
        t.start()
    for t in th:
        t.join()


conc32 = timeit(par32)
ss = [s1, s2] + [rbs.Solver(c.dim, c.m, c.blocks).load_basis(W, A, f) for _ in range(2)]
sts = [st1, st2, torch.cuda.Stream(), torch.cuda.Stream()]
mus4 = query_set(c)[:128]


def parK(K):
    th = [threading.Thread(target=lambda k=k: ss[k].solve_batch(mus4[32 * k:32 * (k + 1)], want_a_n=False,
                                                                stream=sts[k])) for k in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()


for K in (3, 4):
    tK = timeit(lambda: parK(K))
    print(f"{K} x B=32 concurrent: {32 * K / tK:.1f} q/s")
print(f"one B=32: {32/one:.1f} q/s   two B=16 sequential: {32/seq:.1f} q/s   two B=16 concurrent: {32/conc:.1f} q/s"
      f"   two B=32 concurrent: {64/conc32:.1f} q/s")
