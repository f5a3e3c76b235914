"""CPU oracle for the capsule convolution of arXiv 2104.02621.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import this package.  The product package ``paper_2104_02621_b200`` never
imports it and shares no code with it.

The arithmetic lives in ``capsconv_oracle.c`` (plain C, fp64, OpenMP over the
outermost output index); this module only builds it with gcc, marshals numpy
arrays through ctypes and composes single layers into the stack of config 5.

Parity status of every function (see DESIGN.md §3 "Oracle pins"):
  output_dims, fwd, bwd_data, bwd_kernel  -- pinned (tests/test_oracle_pins.py),
                                             incl. their pad > 0 forms (R21)
  fwd/bwd_data/bwd_kernel_slices          -- pinned: slice-wise = the matrix
                                             oracle per slice, Fig 2 rank-3, adjoints
  round_bf16                              -- pinned (torch bf16 cast, exact cases)
  stack_fwd_bwd                           -- composition of pinned layers;
                                             pinned by the depth-1 reduction and
                                             finite differences on a tiny stack
  sgd_update                              -- pinned: hand-computed step
  primary_to_caps / caps_to_primary       -- pinned: inverse pair, channel order
                                             on a one-hot map (reading R25)
  train_step                              -- composition of pinned pieces; its
                                             primary layer pinned to torch conv2d
"""
from .oracle import (  # noqa: F401
    build,
    lib_path,
    output_dims,
    fwd,
    bwd_data,
    bwd_kernel,
    fwd_slices,
    bwd_data_slices,
    bwd_kernel_slices,
    round_bf16,
    num_threads,
    set_num_threads,
    stack_fwd_bwd,
    sgd_update,
    primary_to_caps,
    caps_to_primary,
    train_step,
    OracleError,
)
