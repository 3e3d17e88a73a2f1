"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no prior sampler, no closed-form
convolution, no distance, no selection).  It only produces inputs: frame schedules,
discrepancy weights, input functions, ground-truth phantom TACs (by explicit RK4
integration of the model ODEs, eq:2TCM P:69-80 and the differentiated eq:lp-ntPET
P:84-94 -- a different numerical route from the method's closed forms) and noise
(P:216-220).  Recipes are documented in DESIGN.md ("Input recipe").
"""
from .schedules import (fdg22, tb35, uniform_frames, decay_weights)  # noqa: F401
from .problems import (Problem, config1, config2, config3, config4_chunk, config4_continuous, tb_geometry, tb_voxel_count, brain_geometry, priors_fdg,
                       priors_rt, FENG_PHANTOM)  # noqa: F401
