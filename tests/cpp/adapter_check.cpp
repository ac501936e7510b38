// Compiles the header-only BatchRunner adapter against the C ABI and exercises the paths
// that need no GPU (defaults, nominal pose, structural errors).  Built and run by
// tests/test_cpp_adapter.py.
#include <cmath>
#include <cstdio>

#include "rmpc_b200_batch.hpp"

int main() {
  rmpc_model m = rmpc_b200::default_model();
  rmpc_settings s = rmpc_b200::default_settings(10);
  double q[RMPC_NQ];
  rmpc_nominal_pose(&m, q);
  if (std::fabs(q[1] - 1.0) > 1e-12) return 1;
  try {
    rmpc_b200::BatchRunner bad(0, m, s);
    return 2;
  } catch (const rmpc_b200::Error& e) {
    if (e.code != RMPC_ERR_STRUCTURAL) return 3;
  }
  int code = -1;
  try {
    rmpc_b200::BatchRunner r(8, m, s);
    std::vector<rmpc_state> st(8);
    std::vector<rmpc_command> cm(8, rmpc_command{1.0, 0.0, 0.0});
    std::vector<rmpc_gait> ga(8, rmpc_gait{0.0, 0.8, 1.0, {0.5, 0.5, 0.0, 0.0}});
    for (auto& x : st) for (int k = 0; k < RMPC_NQ; ++k) { x.q[k] = q[k]; x.qd[k] = 0.0; }
    auto out = r.solve(st, cm, ga);
    code = out[0].ok() ? 0 : 4;
  } catch (const rmpc_b200::Error& e) {
    code = e.code == RMPC_ERR_CUDA ? 10 : 5;  // 10: no GPU in this container
  }
  std::printf("%d\n", code);
  return 0;
}
