"""Helpers shared by the tests: golden fixtures and small random instances (no method arithmetic)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def undirected_to_directed(edges):
    """[a, b, act] -> edge 2i = a->b, edge 2i+1 = b->a, both with activation act."""
    src, dst, act = [], [], []
    for a, b, x in edges:
        src += [a, b]
        dst += [b, a]
        act += [x, x]
    return np.array(src, np.uint32), np.array(dst, np.uint32), np.array(act, np.uint8)


def random_instance(rng, n_lo=5, n_hi=30, deg=2.5, amax=8, T_lo=1, T_hi=3, post_hi=3):
    """Random bidirected graph with random activations (activations in [0, 2A])."""
    V = int(rng.integers(n_lo, n_hi + 1))
    m = max(1, int(V * deg / 2))
    u = rng.integers(0, V, m)
    v = rng.integers(0, V, m)
    v = np.where(u == v, (v + 1) % V, v)
    src = np.empty(2 * m, np.uint32)
    dst = np.empty(2 * m, np.uint32)
    src[0::2], dst[0::2] = u, v
    src[1::2], dst[1::2] = v, u
    act = rng.integers(0, amax + 1, 2 * m).astype(np.uint8)
    T = int(rng.integers(T_lo, T_hi + 1))
    terms = [np.unique(rng.integers(0, V, int(rng.integers(1, post_hi + 1)))).astype(np.uint32) for _ in range(T)]
    return V, src, dst, act, terms
