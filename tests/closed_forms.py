"""Closed forms shared by the oracle pins and the GPU tests (test infrastructure: the
mathematics of SURVEY §8.c.3 / [D1], [D4] written out; no method arithmetic of the
CUDA path or of the oracle)."""
import json
import math
import os

import numpy as np

import rbf_workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lattice_constants.json")))
ALPHA, TAIL = GOLD["alias_alpha"], GOLD["tail_t"]
CF_TOL = 3 * 1.7e-9  # SURVEY §8.c.3 / [D4]


def closed_form_gauss(wl, s2):
    """h^2 G_tau(x) / (1 + alpha - t) for f = G_s (unit mass), tau^2 = s^2 - sigma^2."""
    h = wl.meta["h"]
    tau2 = s2 - wl.sigma ** 2
    r2 = wl.xy[:, 0] ** 2 + wl.xy[:, 1] ** 2
    return h * h * np.exp(-r2 / (2 * tau2)) / (2 * math.pi * tau2) / (1 + ALPHA - TAIL)


def closed_form_blobs(wl, seed):
    """f = sum_b a_b exp(-|x - c_b|^2 / 2 s_b^2) = sum_b a_b 2 pi s_b^2 G_{s_b}(x - c_b):
    lambda = h^2 sum_b a_b (s_b^2 / tau_b^2) exp(-|x - c_b|^2 / 2 tau_b^2) / (1 + alpha - t)."""
    h = wl.meta["h"]
    lam = np.zeros(wl.n)
    for c, s, a in zip(*W.blob_params(seed)):
        tau2 = s * s - wl.sigma ** 2
        r2 = (wl.xy[:, 0] - c[0]) ** 2 + (wl.xy[:, 1] - c[1]) ** 2
        lam += a * (s * s / tau2) * np.exp(-r2 / (2 * tau2))
    return h * h * lam / (1 + ALPHA - TAIL)


