/* oracle_abi.h — TEST INFRASTRUCTURE ONLY.  The FP64 per-agent record the CPU checkers
 * (the restated oracle, oracle_capi.cpp, and the reference built from its own sources,
 * oracle/_ref via ref_capi.cpp) return to tests/ and bench.py: MpcSolution's node-0 fields
 * (mpc.hpp:100-116) plus sizes.  Never part of the product ABI. */
#ifndef RMPC_ORACLE_ABI_H_
#define RMPC_ORACLE_ABI_H_
#include <stdint.h>

typedef struct oracle_solution {
  double tau_ff[6], q_set[6], qd_set[6], f0[8], base_residual[3];
  double v_mpc, prim_res, dual_res, delta_inf_norm;
  double v_quad, v_lin;  /* the two terms of V = 1/2 x^T P x + q^T x (cancellation scale) */
  int32_t status, fail_iter, n_vars, n_cons, ldl_nnz, pad;
} oracle_solution;

#endif
