"""Agreement inputs built to hit the corner cases of select_quorum / the
label vote (shared by the CPU oracle-vs-reference test and the GPU sweeps):
NaN and Inf lanes, exactly duplicated replicas (zero distances and diameter
ties between equal-size subsets -> lexicographic tie-break), distances
exactly at epsilon, and argmax ties (first maximum wins)."""
import numpy as np


def adversarial(rng, R, n, v):
    outs = rng.uniform(0, 1, (R, n, v)).round(2)  # coarse values -> many exact ties
    kind = rng.integers(0, 6, R)
    for k in range(R):
        if kind[k] == 0:    # NaN somewhere
            outs[k, rng.integers(n), rng.integers(v)] = np.nan
        elif kind[k] == 1:  # +/-Inf lanes
            outs[k, rng.integers(n), rng.integers(v)] = np.inf
            outs[k, rng.integers(n), rng.integers(v)] = -np.inf
        elif kind[k] == 2:  # duplicated replicas
            src = rng.integers(n)
            outs[k, :] = outs[k, src]
        elif kind[k] == 3:  # two clusters of equal size
            outs[k, : n // 2] = outs[k, 0]
            outs[k, n // 2:] = outs[k, -1]
        elif kind[k] == 4:  # argmax ties inside a row
            outs[k, :, :] = outs[k, 0]
            outs[k, :, 0] = 1.0
            if v > 1:
                outs[k, :, 1] = 1.0
    return outs
