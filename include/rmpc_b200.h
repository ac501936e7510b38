/*
 * rmpc_b200.h — C ABI of the B200-native batched real-time-iteration MPC solver.
 *
 * This is the drop-in boundary for the reference's batched solve entry point
 *   rmpc::BatchRunner(int n_envs, const ModelParams&, const MpcSettings&, int workers)
 *   std::vector<MpcSolution> BatchRunner::solve(states, cmds, gaits, prev, order)
 *   (/root/reference/proj/include/rmpc/batch.hpp:24-46, proj/src/batch.cpp:26-79)
 * and its single-agent twin MpcController::rti_step (proj/include/rmpc/mpc.hpp:137-153).
 *
 * Plain C: POD structs, pointers and sizes; no C++ or torch types in any signature.
 * Inputs are FP64 (the reference's own types); the solve computes in FP32 on sm_100a and
 * returns FP32 solution records.  Per-agent failures never abort the batch: they are
 * reported in rmpc_solution.status, as the reference reports MpcStatus::kFailed
 * (proj/src/mpc.cpp:333-336, batch.hpp:29-31).
 */
#ifndef RMPC_B200_H_
#define RMPC_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RMPC_NQ 9            /* generalized coordinates, robot.hpp:14 */
#define RMPC_NJ 6            /* actuated joints, robot.hpp:15 */
#define RMPC_NC 4            /* contact points (R toe, R heel, L toe, L heel), robot.hpp:16 */
#define RMPC_NF 8            /* contact force components, robot.hpp:17 */
#define RMPC_NV 26           /* decision variables per node (dq, dqd, dF), mpc.hpp:14 */
#define RMPC_MAX_HORIZON 32  /* one warp lane per horizon node during linearization */
#define RMPC_NUM_STAGES 7    /* MpcStage, mpc.hpp:79-88 */

/* ---- return codes of the API calls (structural errors of the reference map here) ---- */
#define RMPC_OK 0
#define RMPC_ERR_STRUCTURAL 1   /* StructuralError: sizes, horizon < 2, length mismatch */
#define RMPC_ERR_INVALID_ARG 2  /* NULL handle / pointer */
#define RMPC_ERR_CUDA 3         /* CUDA runtime failure (no device, launch failure) */
#define RMPC_ERR_NO_KERNEL 4    /* kernel image for this device missing (not sm_100a) */

/* ---- per-agent status codes (MpcStatus + the exception class that caused kFailed) ---- */
#define RMPC_STATUS_OK 0
#define RMPC_STATUS_NONFINITE_INPUT 1  /* StructuralError "build_qp: non-finite linearization point" */
#define RMPC_STATUS_DIVERGED 2         /* DivergenceError "admm: non-finite iterate at iteration k" */
#define RMPC_STATUS_SINGULAR 3         /* SingularityError: non-positive pivot in the factorization */

/* ModelParams (robot.hpp:24-50).  Defaults from rmpc_model_default(). */
typedef struct rmpc_model {
  double torso_mass, torso_len, torso_inertia;
  double thigh_mass, thigh_len, thigh_inertia;
  double shank_mass, shank_len, shank_inertia;
  double foot_mass, foot_half_len, foot_inertia;
  double ankle_drop;
  double joint_lo[RMPC_NJ], joint_hi[RMPC_NJ];
  double qd_limit[RMPC_NJ], tau_limit[RMPC_NJ];
  double kp[RMPC_NJ], kd[RMPC_NJ];
  double mu;        /* model friction (unused by the MPC: it uses settings.mu, mpc.cpp:188) */
  double gravity;
  double nominal_stagger, nominal_drop;
} rmpc_model;

/* MpcSettings (mpc.hpp:16-57) + AdmmSettings::ruiz_iters (qp.hpp:34). */
typedef struct rmpc_settings {
  int32_t horizon;                       /* T, 2 <= T <= RMPC_MAX_HORIZON */
  double dt_schedule[RMPC_MAX_HORIZON];  /* first `horizon` entries used */
  double w_q[RMPC_NQ], w_qd[RMPC_NQ], w_f[RMPC_NF];
  double gait_period, phase_switch, phase_offsets[RMPC_NC];
  double z_swing, v_to, v_td;
  int32_t n_qp;                          /* fixed ADMM iteration count, no early exit */
  double mu, sigma, rho, over_relax;
  int32_t warm_start;                    /* 0: cold nominal guess (default) */
  int32_t ruiz_iters;                    /* 10 (AdmmSettings default, the reference MPC's fixed
                                            value); >= 1 (RMPC_ERR_STRUCTURAL otherwise) */
} rmpc_settings;

/* RobotState (robot.hpp:52-55). */
typedef struct rmpc_state {
  double q[RMPC_NQ];
  double qd[RMPC_NQ];
} rmpc_state;

/* MpcCommand (mpc.hpp:59-63). */
typedef struct rmpc_command {
  double height, vx, wpitch;
} rmpc_command;

/* GaitState (gait.hpp:16-29). */
typedef struct rmpc_gait {
  double phase, period, phase_switch;
  double offsets[RMPC_NC];
} rmpc_gait;

/* MpcSolution (mpc.hpp:100-116), node-0 quantities; z_star is a separate optional array
 * laid out [agent][node][26] = (q 9, qd 9, F 8) per node. */
typedef struct rmpc_solution {
  float tau_ff[RMPC_NJ];
  float q_set[RMPC_NJ];
  float qd_set[RMPC_NJ];
  float f0[RMPC_NF];          /* z_star.F row 0 */
  float base_residual[3];
  float v_mpc;                /* QP objective at the solution step */
  float prim_res, dual_res;
  float delta_inf_norm;       /* ||dz||_inf of the accepted step */
  int32_t status;             /* RMPC_STATUS_* */
  int32_t fail_iter;          /* DivergenceError::iteration, -1 otherwise */
} rmpc_solution;

/* TimingReport (batch.hpp:12-18), measured on the device.  With stage profiling enabled
 * (rmpc_set_stage_profiling), stage_ms splits the fused kernel's time by the reference's 7
 * stages, and stage_mean_ms / stage_std_ms are TimingReport::mean_ms / std_ms: the mean and
 * standard deviation over agents of each agent's time in a stage (clock64 cycles at the
 * reference's stage boundaries, converted at the device's SM clock); else all 0. */
typedef struct rmpc_timing {
  int32_t batch_size;
  int32_t devices;
  double total_ms;     /* wall time of the whole call (host clock) */
  double h2d_ms;       /* host->device copies (max over devices, CUDA events) */
  double kernel_ms;    /* solve kernel (max over devices, CUDA events) */
  double d2h_ms;       /* device->host copies (max over devices, CUDA events) */
  double stage_ms[RMPC_NUM_STAGES];
  double stage_mean_ms[RMPC_NUM_STAGES];
  double stage_std_ms[RMPC_NUM_STAGES];
} rmpc_timing;

typedef struct rmpc_handle rmpc_handle;

void rmpc_model_default(rmpc_model* model);
/* Defaults of MpcSettings with `horizon` nodes of dt = 0.05 (config.cpp:149-151). */
void rmpc_settings_default(rmpc_settings* settings, int32_t horizon);

/* BatchRunner ctor.  Agents are split into contiguous ranges over `devices`
 * (n_devices >= 1; NULL devices = {0}).  Returns RMPC_ERR_STRUCTURAL for n_agents < 1,
 * horizon < 2 or > RMPC_MAX_HORIZON (batch.cpp:19, mpc.cpp:243-245). */
int32_t rmpc_create(const rmpc_model* model, const rmpc_settings* settings, int32_t n_agents,
                    const int32_t* devices, int32_t n_devices, rmpc_handle** out);
void rmpc_destroy(rmpc_handle* handle);

/* BatchRunner::solve with HOST arrays of length n_agents (rmpc_state/command/gait, and
 * optionally prev/prev_z_star for warm start).  Blocks until every device finished (the
 * tick barrier).  Host buffers may be pageable; they are staged through pinned memory.
 * z_star_out may be NULL. */
int32_t rmpc_solve(rmpc_handle* handle, const rmpc_state* states, const rmpc_command* cmds,
                   const rmpc_gait* gaits, const rmpc_solution* prev, const float* prev_z_star,
                   rmpc_solution* out, float* z_star_out);

/* Same solve with DEVICE arrays already resident on the handle's single device; enqueued on
 * `stream` (a cudaStream_t; NULL = the legacy default stream, like every device entry point of
 * the library) without host synchronisation.  Multi-device handles: rmpc_solve_device_sharded. */
int32_t rmpc_solve_device(rmpc_handle* handle, const rmpc_state* d_states,
                          const rmpc_command* d_cmds, const rmpc_gait* d_gaits,
                          const rmpc_solution* d_prev, const float* d_prev_z_star,
                          rmpc_solution* d_out, float* d_z_star_out, void* stream);

/* rmpc_solve_device for a handle over several devices: per shard g (rmpc_shard_info: device,
 * agent range [begin, begin + count) of the batch), its device arrays d_*[g] of `count` agents
 * on that device and streams[g] (NULL array or entry = the device's legacy default stream).
 * d_prev / d_prev_z_star / d_z_star_out may be NULL arrays.  Enqueues one launch per device and
 * returns without host synchronisation; no data crosses devices (agents are independent). */
int32_t rmpc_solve_device_sharded(rmpc_handle* handle, const rmpc_state* const* d_states,
                                  const rmpc_command* const* d_cmds, const rmpc_gait* const* d_gaits,
                                  const rmpc_solution* const* d_prev, const float* const* d_prev_z_star,
                                  rmpc_solution* const* d_out, float* const* d_z_star_out,
                                  void* const* streams);
/* ---- structure-of-arrays boundary (north star: agents laid out SoA for coalesced HBM access) ----
 * The same solve with the per-agent inputs as one FP32 block of RMPC_SOA_FIELDS component rows,
 * row r holding component r of every agent: soa[r * ld + agent], ld >= n_agents.  112 bytes per
 * agent instead of the 224 of the FP64 records.  Row order (the fields of RobotState, MpcCommand
 * and GaitState, robot.hpp:52-55, mpc.hpp:59-63, gait.hpp:16-29): */
#define RMPC_SOA_Q 0              /* q[0..8]       rows 0..8   */
#define RMPC_SOA_QD 9             /* qd[0..8]      rows 9..17  */
#define RMPC_SOA_HEIGHT 18        /* cmd.height */
#define RMPC_SOA_VX 19            /* cmd.vx */
#define RMPC_SOA_WPITCH 20        /* cmd.wpitch */
#define RMPC_SOA_PHASE 21         /* gait.phase */
#define RMPC_SOA_PERIOD 22        /* gait.period */
#define RMPC_SOA_PHASE_SWITCH 23  /* gait.phase_switch */
#define RMPC_SOA_OFFSETS 24       /* gait.offsets[0..3] rows 24..27 */
#define RMPC_SOA_FIELDS 28
/* Each value is widened to FP64 exactly (float -> double), so the result equals rmpc_solve on
 * the FP64 records holding those widened values, bit for bit.  A device kernel unpacks the block
 * with coalesced loads (one thread per agent, consecutive agents on consecutive lanes) into the
 * handle's per-agent records.  Host version: soa may be pageable or pinned, any number of
 * devices (shard g reads columns [begin, begin + count) of every row). */
int32_t rmpc_solve_soa(rmpc_handle* handle, const float* soa, int64_t ld, const rmpc_solution* prev,
                       const float* prev_z_star, rmpc_solution* out, float* z_star_out);
/* Device version (single-device handles): d_soa resident on the handle's device, enqueued on
 * `stream` (NULL = legacy default stream).  Unpacks into the handle's own record buffers, so
 * device solves of one handle must be issued on one stream (as for schedule sharing). */
int32_t rmpc_solve_soa_device(rmpc_handle* handle, const float* d_soa, int64_t ld, const rmpc_solution* d_prev,
                              const float* d_prev_z_star, rmpc_solution* d_out, float* d_z_star_out, void* stream);

/* The agent split of rmpc_create and of one-rank-per-GPU deployments: shard g of G owns
 * [floor(g n / G), floor((g + 1) n / G)).  Host only (no device needed). */
int32_t rmpc_shard_range(int32_t n_agents, int32_t n_shards, int32_t shard, int32_t* begin, int32_t* count);
/* Shard g of the handle: its CUDA device and contiguous agent range. */
int32_t rmpc_shard_info(const rmpc_handle* handle, int32_t shard, int32_t* device, int32_t* begin,
                        int32_t* count);

int32_t rmpc_size(const rmpc_handle* handle);        /* BatchRunner::size() */
int32_t rmpc_workers(const rmpc_handle* handle);     /* BatchRunner::workers(): devices */
int32_t rmpc_horizon(const rmpc_handle* handle);
int32_t rmpc_last_timing(const rmpc_handle* handle, rmpc_timing* out);  /* last_timing() */
const char* rmpc_last_error(const rmpc_handle* handle);  /* NULL handle: creation error */
const char* rmpc_status_message(int32_t status);
const char* rmpc_stage_name(int32_t stage);              /* mpc_stage_name, mpc.cpp:22-26 */

/* Nominal standing pose of the model (robot.cpp:245-306), FP64 host computation. */
void rmpc_nominal_pose(const rmpc_model* model, double q_out[RMPC_NQ]);

/* PD + feed-forward torque from a solution (mpc_torque -> pd_torque, mpc.cpp:340-344,
 * robot.cpp:235-241); returns RMPC_ERR_STRUCTURAL for a failed solution. */
int32_t rmpc_mpc_torque(const rmpc_model* model, const rmpc_solution* sol,
                        const rmpc_state* state, double tau_out[RMPC_NJ]);

/* rmpc_solve_device plus the active set of the final ADMM iterate (the north star's parity
 * criterion): d_active receives n x (horizon + 1) x 40 bytes on the solver's padded row grid
 * (block -1 = the 18 initial-state rows at slots 12..29, then per node: 0..8 integration,
 * 9..11 base dynamics, 12 + 4c + t contact c row t, 28..39 joint boxes), each 0 inactive,
 * 1 at the lower bound, 2 at the upper bound, 3 equality row or no row (all 3 for a failed
 * agent).  Cold start, no z*. */
int32_t rmpc_solve_device_active_set(rmpc_handle* handle, const rmpc_state* d_states,
                                     const rmpc_command* d_cmds, const rmpc_gait* d_gaits,
                                     rmpc_solution* d_out, uint8_t* d_active, void* stream);

/* Schedule-shared factorization (default: level 2).  With warm_start off the QP matrices, the
 * Ruiz scaling and the KKT factor of an agent depend only on its contact schedule (the stance
 * flags of every horizon node; mpc.cpp:266-276 linearizes about the nominal pose), so each solve
 * first hashes every agent's schedule, factorizes each distinct schedule once, and lets every
 * agent of that schedule load the result.  Levels: 0 off (per-agent factorization, also every
 * warm-started solve); 1 one warp pair per agent on the shared factor (bit-identical to 0);
 * 3 squads -- 32 agents of a schedule per warp pair, lane = agent (horizon <= 10; horizons 11..20:
 * long squads of four warps, the half-horizon chains handed between two warps each; beyond: 1);
 * 2 (default) squads where the shard is larger than two waves of the per-agent kernel, else 0
 * (a squad's latency exceeds a small batch's per-agent solve).  Calls on one handle share the
 * schedule workspace: issue device solves of one handle on one stream. */
int32_t rmpc_set_schedule_sharing(rmpc_handle* handle, int32_t enabled);

/* Stage-profiling switch: when on, the kernel samples the SM clock at the reference's stage
 * boundaries and rmpc_last_timing() reports the per-stage split of kernel_ms. */
int32_t rmpc_set_stage_profiling(rmpc_handle* handle, int32_t enabled);

/* Solve-path kernels this process has launched so far (every entry point, every handle):
 * benchmarks difference it over a timed region to count the library's launches. */
int64_t rmpc_kernel_launches(void);

/* Build provenance: "sm_100a" and the kernel variant compiled in. */
const char* rmpc_build_info(void);

/* Measured FP32 FMA throughput of `device` (TFLOP/s): the CUDA-core roofline denominator. */
int32_t rmpc_fma_peak(int32_t device, double* tflops);

/* Dynamic shared memory one agent (one warp pair) needs at `horizon` nodes. */
int32_t rmpc_smem_bytes(int32_t horizon);
/* Agents per CTA (= per SM: one CTA per SM) at `horizon` nodes, bounded by the 512 TMEM columns
 * that hold the factor and the 227 KB of shared memory: 6 warp pairs (384 threads, 168
 * registers) in general, 8 (512 threads, 128 registers) when every node block fits TMEM
 * at 4 warps per lane quarter (horizon <= 8). */
int32_t rmpc_agents_per_cta(int32_t horizon);
/* sizeof of the ABI structs (0 model, 1 settings, 2 state, 3 command, 4 gait, 5 solution,
 * 6 timing) for binding-side layout checks. */
int32_t rmpc_sizeof(int32_t which);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* RMPC_B200_H_ */
