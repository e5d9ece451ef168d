"""Shared helpers for the test suite (unique module name: a foreign `tests`
package is importable in this image)."""


def approx(a, b, eps):
    """doctest::Approx(b).epsilon(eps) semantics: |a-b| < eps*(1 + max(|a|,|b|))."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))
