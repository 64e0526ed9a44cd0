"""B200-native hot path of IGS-GMRES (arXiv 2205.07805): libigs.so (CUDA, sm_100a) behind
the C ABI of include/igs.h, with a thin ctypes binding (igs.py)."""
from .igs import (  # noqa: F401
    EXPORTS, IGS_MEM_DEVICE, IGS_MEM_HOST, KERNEL_KINDS, IgsError, Solver, igs_bind_workspace,
    igs_create, igs_destroy, igs_kernel_stats, igs_nccl_unique_id, igs_op_block_dot, igs_op_spmv,
    igs_op_trisolve, igs_op_update, igs_qr, igs_op_basis_diag, igs_plan_ghosts, igs_plan_remap, igs_plan_sell, igs_result, igs_set_timing,
    igs_solve, igs_solve_alg, igs_stats, igs_workspace_bytes, lib, ALGORITHMS, igs_info, igs_set_timeout,
    igs_bench_block_dot, VirtualGroup,
)
