"""Configuration knobs (mirror of the reference's src/config.py:1-22).

``DEFAULT_VALUE_DTYPE`` / ``DEFAULT_INDEX_DTYPE`` define the parity contract
(8-byte values, 4-byte indices). ``OPALG_DEBUG_CONTRACTS`` keeps the
give-then-use guard of src/ownership.py:37-41 switchable.
"""

import os

DEFAULT_VALUE_DTYPE = "float64"
DEFAULT_INDEX_DTYPE = "int32"

#: raise ContractViolation on use after give() (reference src/config.py:13-15)
debug_contracts = os.environ.get("OPALG_DEBUG_CONTRACTS", "1") != "0"

#: default CUDA device ordinal for CudaExecutor()
DEFAULT_DEVICE = int(os.environ.get("B200SP_DEVICE", "0"))

#: iterations launched per CUDA-graph batch by the device solvers
SOLVER_BATCH = int(os.environ.get("B200SP_SOLVER_BATCH", "16"))

#: unpreconditioned Csr CG up to this many rows runs as one persistent
#: cooperative kernel (0 disables)
CG_COOP_MAX_ROWS = int(os.environ.get("B200SP_CG_COOP_MAX_ROWS", str(1 << 20)))
# GMRES: one single-block launch per Arnoldi step for systems of <= 4096 rows
GMRES_SMALL = os.environ.get("B200SP_GMRES_SMALL", "1") != "0"
# GMRES: systems of <= 4 rows run a whole Arnoldi cycle in one thread, on chip
GMRES_TINY = os.environ.get("B200SP_GMRES_TINY", "1") != "0"
# BiCGSTAB and FCG on the same cooperative single-launch path as CG (same row limit)
BICGSTAB_COOP = os.environ.get("B200SP_BICGSTAB_COOP", "1") != "0"

#: CG / BiCGSTAB on a classical-strategy Csr fuse the reduction after each
#: SpMV into its epilogue (csr_spmv_dot); False runs SpMV + dot kernels
FUSED_SPMV_DOT = os.environ.get("B200SP_FUSED_SPMV_DOT", "1") != "0"
# distributed CG halo: "auto" = peer memory (CUDA IPC) under NCCL when every
# send is a row range, "1" = force it (also over gloo: ranks sharing one GPU),
# "0" = NCCL send/recv
PEER_HALO = os.environ.get("B200SP_PEER_HALO", "auto")
# distributed CG: capture a batch of iterations as a CUDA graph when the halo
# and the all-reduces both go through peer memory (no host collective inside)
DIST_GRAPH = os.environ.get("B200SP_DIST_GRAPH", "1") != "0"
