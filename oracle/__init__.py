"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference rasterizer path
(/root/reference/pkg/src/tilesplat), used ONLY by tests/, by
__graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
`--impl reference` leg.  The product package `paper_2601_19489_b200` never
imports it; its only implementation is the CUDA library.

Parity is PINNED: tests/test_oracle_golden.py checks every function here
against golden vectors produced by the unmodified reference
(tests/golden/make_golden.py imports tilesplat from /root/reference).
"""

from .raster import (adam_step, backward_per_gaussian, bin_load_balanced, bin_sequential,
                     make_scene, photometric, project, project_vjp, render, snugboxes)

__all__ = ["adam_step", "backward_per_gaussian", "bin_load_balanced", "bin_sequential",
           "make_scene", "photometric", "project", "project_vjp", "render", "snugboxes"]
