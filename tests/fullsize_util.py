"""Shared checks of the full-size GPU parity tests against the recorded CPU
oracle runs (tools/oracle_fullsize.py).

State evidence at every step:
* full-state 2-norms (``u_norm``/``v_norm``);
* a Johnson–Lindenstrauss estimate of the FULL-state relative L2 error: the
  fixture holds g_k·u and h_k·v for K seeded Gaussian vectors, and
  (1/K) Σ_k [(g_k·Δu)² + (h_k·Δv)²] is an unbiased estimate of ‖Δu‖² + ‖Δv‖²
  (≥ 32 χ² degrees of freedom: the estimate stays within ×[0.5, 1.6] of the
  truth with probability > 0.999);
* at the steps in ``sub_steps``: the exact rel-L2 on a stride-``sub_stride``
  subsample of u and v.
"""
import json
import os

import numpy as np

from conftest import GOLDEN


def load(name):
    """(fixture dict, {'u_<step>': …, 'v_<step>': …} or {})."""
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        return None, None
    ref = json.load(open(path))
    sf = ref.get("states_file")
    states = {}
    if sf and os.path.exists(os.path.join(GOLDEN, sf)):
        states = dict(np.load(os.path.join(GOLDEN, sf)))
    return ref, states


class StateChecker:
    def __init__(self, ref, states):
        self.ref, self.states = ref, states
        self.k = int(ref.get("proj_k", 0))
        if self.k:
            rng = np.random.default_rng(int(ref["proj_seed"]))
            self.gu = rng.standard_normal((self.k, ref["n"]))
            self.gv = rng.standard_normal((self.k, ref["m"]))
        self.worst_proj = 0.0
        self.worst_sub = 0.0

    def check(self, step, u, v, bound=1e-8):
        """step is 1-based; u, v numpy fp64 full states."""
        ref, j = self.ref, step - 1
        assert abs(np.linalg.norm(u) / ref["u_norm"][j] - 1) <= bound, ("u_norm", step)
        assert abs(np.linalg.norm(v) / ref["v_norm"][j] - 1) <= bound, ("v_norm", step)
        if self.k:
            du = self.gu @ u - np.asarray(ref["u_proj"][j])
            dv = self.gv @ v - np.asarray(ref["v_proj"][j])
            est = np.sqrt((np.sum(du ** 2) + np.sum(dv ** 2)) / self.k) / np.sqrt(
                ref["u_norm"][j] ** 2 + ref["v_norm"][j] ** 2)
            self.worst_proj = max(self.worst_proj, est)
            assert est <= bound, ("projected rel-L2", step, est)
        if f"u_{step}" in self.states:
            s = ref["sub_stride"]
            ru, rv = self.states[f"u_{step}"], self.states[f"v_{step}"]
            gu, gv = u[::s], v[::s]
            rel = np.sqrt(np.sum((gu - ru) ** 2) + np.sum((gv - rv) ** 2)) / np.sqrt(
                np.sum(ru ** 2) + np.sum(rv ** 2))
            self.worst_sub = max(self.worst_sub, rel)
            assert rel <= bound, ("subsample rel-L2", step, rel)
