"""Break-even density of a sparse kernel against a dense one.

P:L505 [§Evaluation]: "The use of a sparse convolution is not always profitable.
Above certain density levels, a dense convolution implementation is more
profitable than the sparse counterpart ... the break-even density level (43.5%)".
Given sparse times measured at increasing densities and one dense time, the
break-even density is where the sparse time curve reaches the dense time.
Host-side arithmetic only (no GPU); ``scripts/breakeven.py`` supplies timings.
"""
from __future__ import annotations


def break_even_density(densities, sparse_times, dense_time):
    """Smallest density at which the sparse time reaches ``dense_time``.

    ``densities`` must be strictly increasing.  Linear interpolation between the
    two sweep points that bracket the crossing; the first point is returned if the
    sparse kernel is already slower there; ``None`` if it is faster everywhere.
    """
    d = list(densities)
    t = list(sparse_times)
    if len(d) != len(t) or not d:
        raise ValueError("densities and times must be non-empty and of equal length")
    if any(b <= a for a, b in zip(d, d[1:])):
        raise ValueError("densities must be strictly increasing")
    if t[0] >= dense_time:
        return d[0]
    for i in range(1, len(d)):
        if t[i] >= dense_time:
            frac = (dense_time - t[i - 1]) / (t[i] - t[i - 1])
            return d[i - 1] + frac * (d[i] - d[i - 1])
    return None
