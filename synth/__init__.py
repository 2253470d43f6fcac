"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module holds NO arithmetic of the method (no domain transform, no filter,
no solver step).  It only draws guides, targets and confidences.  It is the one
module both the oracle side (tests, bench cpu_baseline) and the CUDA side
(tests, bench) use, so that both see bit-identical fp32 inputs.  Recipes are in
DESIGN.md "Input recipe"; unstated details are our choices.
"""
from .configs import CONFIGS, Config, make_inputs, random_problem, target_range  # noqa: F401
