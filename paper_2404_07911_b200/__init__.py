"""paper_2404_07911_b200 — B200-native matrix-free DG-CutFEM operator apply.

Thin Python binding (argument marshalling only) over the C ABI in
``include/cutfem.h`` implemented by ``libcutfem.so`` (hand-written sm_100a
FP64 kernels).  Every step of v = A u runs in the CUDA kernels; there is no
CPU fallback: if the shared library is missing or no CUDA device is present,
calls raise.

Method: PAPER.md (arXiv 2404.07911) §3 "Matrix-free implementation"; see
DESIGN.md for the kernels, the data layout and the readings of the paper.
"""
from ._lib import (CutFEM, CutFEMDist, CutFEMH1, CutFEMMG, LocalProblem, TERM_ALL, TERM_CELL, TERM_GP,  # noqa: F401
                   TERM_NITSCHE, TERM_SIPG, build, lib_path, load, nccl_unique_id, partition_x)

__all__ = ["CutFEM", "CutFEMDist", "CutFEMH1", "CutFEMMG", "LocalProblem", "partition_x", "nccl_unique_id", "build", "load", "lib_path", "TERM_ALL", "TERM_CELL", "TERM_SIPG",
           "TERM_NITSCHE", "TERM_GP"]
