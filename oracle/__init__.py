"""TEST INFRASTRUCTURE ONLY -- float64 CPU oracle for the paper's discrete A and A*.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2510_24687_b200``) never imports, links or executes it, and this package
never imports the product path.  The only module both sides share is ``synth``
(seeded input generators, no method arithmetic).
"""
from .tat_oracle import (  # noqa: F401
    Constants, derive, forward, adjoint, forward_stages, adjoint_stages,
    cartesian_spectrum, polar_resample, angular_coefficients, multiplier_table,
    apply_multiplier, cosine_transform, synthesis, restrict,
)
