/*
 * rmpc_b200_env.h — C ABI of the closed-loop step that follows the batched solve
 * (SURVEY.md §8(f) rows 1-2), device-resident and asynchronous on a CUDA stream:
 *
 *   rmpc_physics_step_device   physics_step      (/root/reference/proj/src/env.cpp:38-68):
 *                              penalty contacts on the terrain, `substeps` semi-implicit
 *                              Euler steps with qdd = M^-1 (tau - h + J^T F) (LLT), then
 *                              advance_phase (gait.cpp:31-35)
 *   rmpc_control_step_device   mpc_torque + blend + physics_step fused in one kernel
 *                              (mpc.cpp:340-344, policy.cpp:133-157, ppo.cpp:345-349): the
 *                              torque a failed solution yields is zero, as in Trainer::train
 *   rmpc_observe_device        observe (policy.cpp:104-122): the 23-entry policy input
 *   rmpc_policy_forward_device policy_forward (policy.cpp:85-102): the residual MLPs
 *   rmpc_ppo_*, rmpc_gae_device, rmpc_adam_*
 *                              the PPO batch (ppo.cpp:28-276): loss + gradient, GAE, Adam,
 *                              whole ppo_update calls on a device-resident rollout
 *
 * The environment owns the reference's EnvConfig physics/terrain part (env.hpp:52-63) and the
 * heightfield (Terrain, env.cpp:8-27, drawn from Rng(seed, 0x7e22) like the reference).  Each
 * agent carries its randomize_model draw (env.cpp:196-208) as rmpc_body {mu, mass_scale};
 * a NULL body array means the base model.  All arithmetic is FP64 (the simulator's state
 * integrates over thousands of steps).  Per-agent blow-ups never abort the batch: status 1
 * replaces the reference's SimBlowupError.
 */
#ifndef RMPC_B200_ENV_H_
#define RMPC_B200_ENV_H_

#include "rmpc_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define RMPC_OBS_DIM 23

/* EnvConfig (env.hpp:52-63) and TerrainConfig (env.hpp:16-23). */
typedef struct rmpc_env_config {
  double control_dt;     /* 0.01 s (100 Hz control) */
  int32_t substeps;      /* 4 (400 Hz physics) */
  int32_t terrain_kind;  /* 0 flat, 1 heightfield */
  double k_n, c_n, v_slip;           /* penalty contact: 5e4, 500, 0.05 */
  double amplitude, cell, extent;    /* heightfield: 0.04, 0.3, 80 */
  uint64_t terrain_seed;             /* 0 */
} rmpc_env_config;

/* randomize_model (env.cpp:196-208): friction and one common mass/inertia scale. */
typedef struct rmpc_body {
  double mu;
  double mass_scale;
} rmpc_body;

/* BlendStrategy (policy.hpp): joint-joint, joint-torque, torque-torque (policy.cpp:133-157). */
enum {
  RMPC_BLEND_JOINT_JOINT = 0,
  RMPC_BLEND_JOINT_TORQUE = 1,
  RMPC_BLEND_TORQUE_TORQUE = 2
};

/* Simulation outcome per agent. */
enum { RMPC_SIM_OK = 0, RMPC_SIM_BLOWUP = 1 };

typedef struct rmpc_env rmpc_env;

void rmpc_env_config_default(rmpc_env_config* cfg);
/* Builds the terrain on the host and uploads it with the base model to `device`. */
int32_t rmpc_env_create(const rmpc_model* base, const rmpc_env_config* cfg, int32_t device,
                        rmpc_env** out);
void rmpc_env_destroy(rmpc_env* env);
/* Terrain::height_at (env.cpp:17-27) on the host copy, for tests and callers. */
int32_t rmpc_env_height_at(const rmpc_env* env, double x, double* h);

/* One control period for n agents.  states/gaits are updated in place; tau is n x 6 (FP64);
 * sim_status (n, may be NULL) receives RMPC_SIM_*.  stream 0 = the legacy default stream. */
int32_t rmpc_physics_step_device(rmpc_env* env, int32_t n, rmpc_state* d_states,
                                 rmpc_gait* d_gaits, const rmpc_body* d_bodies,
                                 const double* d_tau, int32_t* d_sim_status, void* stream);

/* tau = blend(mpc_torque(sol), ...) (zero for a failed solution), then the physics step.
 * d_action (n x 6) may be NULL (zero action); d_tau_out (n x 6) may be NULL. */
int32_t rmpc_control_step_device(rmpc_env* env, int32_t n, const rmpc_solution* d_sol,
                                 const double* d_action, int32_t strategy, double lambda,
                                 rmpc_state* d_states, rmpc_gait* d_gaits,
                                 const rmpc_body* d_bodies, double* d_tau_out,
                                 int32_t* d_sim_status, void* stream);

/* observe(state, solution) -> n x RMPC_OBS_DIM FP64 (ObsSettings: v_mpc_scale 1e-2,
 * v_mpc_sentinel 10 for a failed solution). */
int32_t rmpc_observe_device(int32_t n, const rmpc_state* d_states, const rmpc_gait* d_gaits,
                            const rmpc_solution* d_sol, double v_mpc_scale,
                            double v_mpc_sentinel, double* d_obs, void* stream);

/* Plan feedback for open-loop replanning benchmarks: state <- node 1 of
 * the previous plan z* (q*[1], qd*[1]; n x horizon x 26 FP32 as rmpc_solve writes it), gait
 * phase advanced by dt (advance_phase, gait.cpp:31-35).  Agents whose solve failed keep their
 * state and only advance the phase. */
int32_t rmpc_plan_feedback_device(int32_t n, int32_t horizon, const float* d_z,
                                  const rmpc_solution* d_sol, rmpc_state* d_states,
                                  rmpc_gait* d_gaits, double dt, void* stream);

/* Residual policy forward: policy_forward (policy.cpp:85-102) for n
 * agents, FP64 like the reference: two 4-layer ELU MLPs (obs -> hidden -> hidden -> hidden ->
 * act / 1).  `params` is MlpParams::flatten_into order (policy.cpp:40-47) of pi then value --
 * per layer W (out x in, column-major as Eigen stores it) then b -- then log_std (act_dim):
 * n_params = pi.num_params() + value.num_params() + act_dim (PolicyParams::num_params). */
typedef struct rmpc_policy rmpc_policy;
int32_t rmpc_policy_create(int32_t obs_dim, int32_t act_dim, int32_t hidden, const double* params,
                           int32_t n_params, int32_t device, rmpc_policy** out);
void rmpc_policy_destroy(rmpc_policy* policy);
/* mean (n x act_dim) and value (n); either output may be NULL. */
int32_t rmpc_policy_forward_device(rmpc_policy* policy, int32_t n, const double* d_obs,
                                   double* d_mean, double* d_value, void* stream);

/* Parameter count (pi + value + log_std, PolicyParams::num_params) and host copies of the
 * device parameters in flatten_policy order (ppo.cpp:144-162). */
int32_t rmpc_policy_num_params(const rmpc_policy* policy);
int32_t rmpc_policy_get_params(rmpc_policy* policy, double* params, int32_t n_params);
int32_t rmpc_policy_set_params(rmpc_policy* policy, const double* params, int32_t n_params);

/* ---- PPO batch (/root/reference/proj/src/ppo.cpp:28-276), FP64. ---- */

/* PpoConfig (ppo.hpp:14-24), the update part. */
typedef struct rmpc_ppo_config {
  double gamma, lam_gae, clip_eps;   /* 0.99, 0.95, 0.2 */
  int32_t epochs, minibatches;       /* 4, 4 */
  double lr, entropy_coef, value_coef, max_grad_norm;  /* 3e-4, 0, 0.5, 1 */
} rmpc_ppo_config;
/* PpoLossInfo (ppo.hpp:70-75) and PpoUpdateStats (ppo.hpp:103-108). */
typedef struct rmpc_ppo_loss_info {
  double total, surrogate, value_loss, entropy;
} rmpc_ppo_loss_info;
typedef struct rmpc_ppo_update_stats {
  double loss, surrogate, value_loss, entropy;
} rmpc_ppo_update_stats;

void rmpc_ppo_config_default(rmpc_ppo_config* cfg);

/* ppo_loss (ppo.cpp:79-135) over n samples (obs n x obs_dim, actions n x act_dim, old_logp /
 * advantages / returns n; device pointers): the loss terms into d_info (device, one struct) and,
 * if d_grads is non-NULL, the gradient of every parameter in flatten_grads order
 * (rmpc_policy_num_params doubles, overwritten).  Deterministic: a fixed-order reduction.
 * Calls on one policy share its device workspace: issue them on one stream (or synchronise). */
int32_t rmpc_ppo_loss_device(rmpc_policy* policy, int32_t n, const double* d_obs,
                             const double* d_actions, const double* d_old_logp,
                             const double* d_advantages, const double* d_returns,
                             const rmpc_ppo_config* cfg, double* d_grads,
                             rmpc_ppo_loss_info* d_info, void* stream);

/* gae_advantages (ppo.cpp:28-45): steps x envs row-major, raw (unnormalised) advantages and
 * returns. */
int32_t rmpc_gae_device(int32_t steps, int32_t envs, const double* d_rewards, const double* d_values,
                        const double* d_dones, const double* d_bootstrap, double gamma, double lam,
                        double* d_advantages, double* d_returns, void* stream);

/* AdamOptimizer(num_params, lr) (ppo.cpp:179-193, betas 0.9 / 0.999, eps 1e-8) bound to a
 * policy: its moment vectors live on the policy's device. */
typedef struct rmpc_adam rmpc_adam;
int32_t rmpc_adam_create(rmpc_policy* policy, double lr, rmpc_adam** out);
void rmpc_adam_destroy(rmpc_adam* adam);

/* Rng(seed, stream) (rng.hpp:15-25) as its four xoshiro256++ words, for rmpc_ppo_update_device. */
void rmpc_rng_seed(uint64_t seed, uint64_t stream, uint64_t state[4]);

/* ppo_update (ppo.cpp:195-276) on the policy's device parameters: GAE, advantage
 * normalisation, then epochs x minibatches of {shuffle (Fisher-Yates on rng_state, advanced
 * exactly like the reference's update_rng), ppo_loss + gradient, clip to max_grad_norm, Adam}.
 * The rollout is device-resident, steps x envs (obs steps x envs x obs_dim, actions
 * steps x envs x act_dim).  Blocks until done; stats on the host. */
int32_t rmpc_ppo_update_device(rmpc_policy* policy, rmpc_adam* adam, int32_t steps, int32_t envs,
                               const double* d_obs, const double* d_actions, const double* d_logp,
                               const double* d_values, const double* d_rewards, const double* d_dones,
                               const double* d_bootstrap, const rmpc_ppo_config* cfg,
                               uint64_t rng_state[4], rmpc_ppo_update_stats* stats, void* stream);

/* Measured FP64 FMA throughput of `device` (TFLOP/s): the PPO batch's roofline denominator. */
int32_t rmpc_fma_peak_f64(int32_t device, double* tflops);

/* sizeof of the env ABI structs (0 config, 1 body, 2 ppo config, 3 loss info, 4 update stats)
 * for binding-side layout checks. */
int32_t rmpc_env_sizeof(int32_t which);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* RMPC_B200_ENV_H_ */
