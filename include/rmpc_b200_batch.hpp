// rmpc_b200_batch.hpp — header-only C++ adapter over the C ABI (rmpc_b200.h) with the method
// names and argument order of rmpc::BatchRunner (/root/reference/proj/include/rmpc/batch.hpp:24-46):
//
//   rmpc_b200::BatchRunner runner(n_envs, model, settings, workers);   // workers = GPUs
//   std::vector<rmpc_b200::Solution> out = runner.solve(states, cmds, gaits, &prev, &order);
//   runner.size(); runner.workers(); runner.last_timing();
//
// Errors the reference throws as StructuralError (batch.cpp:19, 32-36) are thrown here as
// rmpc_b200::Error; per-agent numerical failures are reported in Solution::status and never
// throw (mpc.cpp:333-336).  When the reference's Eigen-typed headers are on the include path
// (RMPC_B200_WITH_REFERENCE_TYPES), solve() also accepts std::vector<rmpc::RobotState> etc.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "rmpc_b200.h"

namespace rmpc_b200 {

struct Error : std::runtime_error {
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
  int code;
};

// MpcSolution (mpc.hpp:100-116): the node-0 record plus z* (T x 26, q | qd | F per node).
struct Solution {
  rmpc_solution rec;
  std::vector<float> z_star;
  bool ok() const { return rec.status == RMPC_STATUS_OK; }
  std::string message() const { return rmpc_status_message(rec.status); }
};

inline rmpc_model default_model() {
  rmpc_model m;
  rmpc_model_default(&m);
  return m;
}

inline rmpc_settings default_settings(int horizon = 12) {
  rmpc_settings s;
  rmpc_settings_default(&s, horizon);
  return s;
}

class BatchRunner {
 public:
  // workers <= 0: one GPU (device 0); workers = k: devices 0..k-1 (agents split contiguously)
  BatchRunner(int n_envs, const rmpc_model& model, const rmpc_settings& settings, int workers = 0)
      : horizon_(settings.horizon) {
    std::vector<int32_t> devs;
    for (int d = 0; d < (workers > 0 ? workers : 1); ++d) devs.push_back(d);
    const int32_t rc = rmpc_create(&model, &settings, n_envs, devs.data(), (int32_t)devs.size(), &h_);
    if (rc != RMPC_OK) throw Error(rc, rmpc_last_error(nullptr));
  }
  BatchRunner(const BatchRunner&) = delete;
  BatchRunner& operator=(const BatchRunner&) = delete;
  ~BatchRunner() { rmpc_destroy(h_); }

  // BatchRunner::solve.  `order` only permutes processing in the reference; results never
  // depend on it (batch.hpp:20-23), so it is validated for length and otherwise ignored.
  std::vector<Solution> solve(const std::vector<rmpc_state>& states,
                              const std::vector<rmpc_command>& cmds,
                              const std::vector<rmpc_gait>& gaits,
                              const std::vector<Solution>* prev = nullptr,
                              const std::vector<int>* order = nullptr, bool want_z = true) {
    const size_t n = (size_t)size();
    if (states.size() != n || cmds.size() != n || gaits.size() != n)
      throw Error(RMPC_ERR_STRUCTURAL, "BatchRunner::solve: input lengths != n_envs");
    if (prev && prev->size() != n) throw Error(RMPC_ERR_STRUCTURAL, "BatchRunner::solve: prev length != n_envs");
    if (order && order->size() != n) throw Error(RMPC_ERR_STRUCTURAL, "BatchRunner::solve: order length != n_envs");
    const size_t zrow = (size_t)horizon_ * RMPC_NV;
    std::vector<rmpc_solution> recs(n);
    std::vector<float> z(want_z ? n * zrow : 0);
    std::vector<rmpc_solution> prev_recs;
    std::vector<float> prev_z;
    if (prev) {
      prev_recs.resize(n);
      prev_z.assign(n * zrow, 0.f);
      for (size_t i = 0; i < n; ++i) {
        prev_recs[i] = (*prev)[i].rec;
        if ((*prev)[i].z_star.size() == zrow)
          std::copy((*prev)[i].z_star.begin(), (*prev)[i].z_star.end(), prev_z.begin() + i * zrow);
        else
          prev_recs[i].status = RMPC_STATUS_NONFINITE_INPUT;  // no z*: not warm-startable
      }
    }
    const int32_t rc = rmpc_solve(h_, states.data(), cmds.data(), gaits.data(),
                                  prev ? prev_recs.data() : nullptr, prev ? prev_z.data() : nullptr,
                                  recs.data(), want_z ? z.data() : nullptr);
    if (rc != RMPC_OK) throw Error(rc, rmpc_last_error(h_));
    std::vector<Solution> out(n);
    for (size_t i = 0; i < n; ++i) {
      out[i].rec = recs[i];
      if (want_z) out[i].z_star.assign(z.begin() + i * zrow, z.begin() + (i + 1) * zrow);
    }
    return out;
  }

  int size() const { return rmpc_size(h_); }
  int workers() const { return rmpc_workers(h_); }
  rmpc_timing last_timing() const {
    rmpc_timing t;
    rmpc_last_timing(h_, &t);
    return t;
  }
  rmpc_handle* handle() const { return h_; }

 private:
  rmpc_handle* h_ = nullptr;
  int horizon_ = 0;
};

}  // namespace rmpc_b200

#if defined(RMPC_B200_WITH_REFERENCE_TYPES) && __has_include(<Eigen/Dense>)
#include "rmpc/batch.hpp"
namespace rmpc_b200 {
// Converters from the reference's Eigen-typed structs (robot.hpp:52-55, mpc.hpp:59-63,
// gait.hpp:16-29) to the C ABI records.
inline rmpc_state to_c(const rmpc::RobotState& s) {
  rmpc_state c;
  for (int k = 0; k < RMPC_NQ; ++k) { c.q[k] = s.q[k]; c.qd[k] = s.qd[k]; }
  return c;
}
inline rmpc_command to_c(const rmpc::MpcCommand& m) { return rmpc_command{m.height, m.vx, m.wpitch}; }
inline rmpc_gait to_c(const rmpc::GaitState& g) {
  rmpc_gait c{g.phase, g.period, g.phase_switch, {g.offsets[0], g.offsets[1], g.offsets[2], g.offsets[3]}};
  return c;
}
}  // namespace rmpc_b200
#endif
