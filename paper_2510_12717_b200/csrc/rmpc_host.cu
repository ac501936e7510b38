// rmpc_host.cu — host runtime behind the C ABI (include/rmpc_b200.h).
//
// BatchRunner (/root/reference/proj/src/batch.cpp:17-79) becomes a handle owning, per device,
// a contiguous agent shard, a stream, device buffers and pinned staging buffers.  A solve
// enqueues H2D copies, the fused kernel and D2H copies on every shard's stream (one host
// thread per device when several are used) and blocks until all shards finished: the tick
// barrier of SPEC.md's batch_runtime.  There is no collective: agents are independent.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rmpc_device.cuh"

namespace {

thread_local std::string g_create_error;
constexpr size_t kSchedCap = 1024;  // distinct schedules stored per shard and tick

struct Shard {
  int device = 0;
  int begin = 0, count = 0;
  int sms = 148;
  cudaStream_t stream = nullptr, stream2 = nullptr;  // stream2: the second chunk of a tick
  cudaEvent_t ev[8] = {};
  rmpc_state* d_states = nullptr;
  rmpc_command* d_cmds = nullptr;
  rmpc_gait* d_gaits = nullptr;
  rmpc_solution* d_prev = nullptr;
  float* d_prev_z = nullptr;
  rmpc_solution* d_out = nullptr;
  float* d_z = nullptr;
  float* d_soa = nullptr;  // rmpc_solve_soa: the shard's FP32 component rows
  unsigned long long* d_prof = nullptr;
  RmpcSchedBuffers sched[1] = {};  // schedule-shared workspace
  // pinned staging for pageable caller buffers
  char* h_stage_in = nullptr;
  char* h_stage_out = nullptr;
  size_t stage_in_bytes = 0, stage_out_bytes = 0;
  double h2d_ms = 0, kernel_ms = 0, d2h_ms = 0;
  unsigned long long prof[2 * RMPC_NUM_STAGES] = {0};  // per stage: sum, then sum of squares
  int clock_khz = 0;
  int err = 0;
  std::string msg;
};

// Persistent host workers for shards 1..G-1 (the calling thread runs shard 0): the reference's
// BatchRunner spawns min(workers, n) threads per solve (batch.cpp:46-62); a control tick every
// 10 ms should not pay thread creation, so the workers live as long as the handle.
class ShardPool {
 public:
  explicit ShardPool(int workers) {
    for (int g = 1; g <= workers; ++g) threads_.emplace_back([this, g]() { loop(g); });
  }
  ~ShardPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  // job(g) for g = 0..G-1, g = 0 on the caller; returns when all are done
  void run(const std::function<void(int)>& job) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      pending_ = (int)threads_.size();
      ++epoch_;
    }
    cv_.notify_all();
    job(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this]() { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int g) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&]() { return stop_ || epoch_ != seen; });
        if (stop_) return;
        seen = epoch_;
        job = job_;
      }
      (*job)(g);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t epoch_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

}  // namespace

struct rmpc_handle {
  rmpc_model model;
  rmpc_settings settings;
  int n = 0;
  int NT = 0;
  double nominal[RMPC_NQ];
  std::vector<Shard> shards;
  rmpc_timing timing;
  std::string err;
  int profile = 0;
  int share = 2;  // cold-start schedule sharing: 0 off, 1 warp-pair CTAs, 2 auto, 3 squads
  std::unique_ptr<ShardPool> pool;  // shards >= 2 only
};

namespace {

// ---------------------------------------------------------------- host model helpers (FP64)
struct P2 {
  double x, z;
};

// Standing pose (robot.cpp:245-306): per-leg 2-link IK for a flat foot with the ankles at
// +-stagger around a shift that is iterated until the CoM is over the contact centroid.
void nominal_pose_host(const rmpc_model& p, double q[RMPC_NQ]) {
  auto leg = [&](double x_off, double out[3]) {
    const double l1 = p.thigh_len, l2 = p.shank_len;
    const double r = std::hypot(x_off, p.nominal_drop);
    const double ck = std::min(1.0, std::max(-1.0, (r * r - l1 * l1 - l2 * l2) / (2.0 * l1 * l2)));
    const double knee = std::acos(ck);
    const double thigh = std::atan2(x_off, p.nominal_drop) - std::atan2(l2 * std::sin(knee), l1 + l2 * std::cos(knee));
    out[0] = thigh;
    out[1] = knee;
    out[2] = -(thigh + knee);
  };
  const double m[7] = {p.torso_mass, p.thigh_mass, p.shank_mass, p.foot_mass,
                       p.thigh_mass, p.shank_mass, p.foot_mass};
  double shift = 0.0;
  for (int it = 0; it < 60; ++it) {
    double L[3], R[3];
    leg(shift + p.nominal_stagger, L);
    leg(shift - p.nominal_stagger, R);
    q[0] = 0.0;
    q[1] = p.ankle_drop + p.nominal_drop + 0.5 * p.torso_len;
    q[2] = 0.0;
    for (int k = 0; k < 3; ++k) { q[3 + k] = L[k]; q[6 + k] = R[k]; }
    // CoM x of the 7 links at zero velocity
    const P2 hip{0.0, q[1] - 0.5 * p.torso_len};
    double cx = m[0] * 0.0, tot = m[0];
    for (int lg = 0; lg < 2; ++lg) {
      const double* a = lg == 0 ? L : R;
      const double a1 = a[0], a2 = a1 + a[1], a3 = a2 + a[2];
      auto pt = [](P2 f, double ang, double x, double z) {
        return P2{f.x + std::cos(ang) * x - std::sin(ang) * z, f.z + std::sin(ang) * x + std::cos(ang) * z};
      };
      const P2 knee = pt(hip, a1, 0.0, -p.thigh_len);
      const P2 ankle = pt(knee, a2, 0.0, -p.shank_len);
      cx += m[1] * pt(hip, a1, 0.0, -0.5 * p.thigh_len).x;
      cx += m[2] * pt(knee, a2, 0.0, -0.5 * p.shank_len).x;
      cx += m[3] * pt(ankle, a3, 0.0, -p.ankle_drop).x;
      tot += m[1] + m[2] + m[3];
    }
    cx /= tot;
    if (std::abs(cx - shift) < 1e-14) break;
    shift = cx;
  }
}

rmpc_dev::KParams make_params(const rmpc_handle& h) {
  rmpc_dev::KParams P;
  std::memset(&P, 0, sizeof(P));
  const rmpc_settings& s = h.settings;
  const rmpc_model& m = h.model;
  P.NT = s.horizon;
  P.n_qp = s.n_qp;
  P.ruiz_iters = s.ruiz_iters;
  P.warm_start = s.warm_start;
  for (int i = 0; i < RMPC_MAX_HORIZON; ++i) P.dt[i] = s.dt_schedule[i];
  for (int k = 0; k < RMPC_NQ; ++k) { P.wq[k] = s.w_q[k]; P.wqd[k] = s.w_qd[k]; P.nominal[k] = h.nominal[k]; }
  for (int k = 0; k < RMPC_NF; ++k) P.wf[k] = s.w_f[k];
  P.z_swing = s.z_swing; P.v_to = s.v_to; P.v_td = s.v_td;
  P.mu = s.mu; P.sigma = s.sigma; P.rho = s.rho; P.alpha = s.over_relax;
  const double ml[7] = {m.torso_mass, m.thigh_mass, m.shank_mass, m.foot_mass, m.thigh_mass, m.shank_mass, m.foot_mass};
  const double il[7] = {m.torso_inertia, m.thigh_inertia, m.shank_inertia, m.foot_inertia,
                        m.thigh_inertia, m.shank_inertia, m.foot_inertia};
  for (int l = 0; l < 7; ++l) { P.m_link[l] = ml[l]; P.I_link[l] = il[l]; }
  P.torso_len = m.torso_len; P.thigh_len = m.thigh_len; P.shank_len = m.shank_len;
  P.foot_half = m.foot_half_len; P.ankle_drop = m.ankle_drop; P.gravity = m.gravity;
  for (int j = 0; j < RMPC_NJ; ++j) { P.jlo[j] = m.joint_lo[j]; P.jhi[j] = m.joint_hi[j]; P.qdlim[j] = m.qd_limit[j]; }
  double tm = 0.0;
  for (double v : ml) tm += v;
  P.weight = tm * m.gravity;
  P.profile = h.profile;
  return P;
}

// The solve path of the handle (rmpc_set_schedule_sharing): 0 per-agent, 1 shared warp pairs,
// 2 squads.  Level 2 ("auto") picks the per-agent kernel when the batch fits two of its waves on
// one device: a squad's latency (~0.6 ms at N = 10) is ~2.5 per-agent waves, so below that the
// per-agent kernel finishes first (C1: 0.21 vs 0.75 ms).  Decided on the whole batch, so every
// shard of a multi-device handle runs the same path (results never depend on the sharding).
// Level 3 forces squads.
int solve_path(const rmpc_handle& h, int sms, bool cold = false) {
  if ((h.settings.warm_start && !cold) || h.share == 0) return 0;
  if (h.share == 1) return 1;
  if (h.share == 2 && h.n <= 2 * sms * rmpc_dev::cta_shape(h.NT).agents) return 0;
  return 2;
}

#define CK(expr)                                                   \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) {                                       \
      sh.err = RMPC_ERR_CUDA;                                      \
      sh.msg = std::string(#expr) + ": " + cudaGetErrorString(e_); \
      return;                                                      \
    }                                                              \
  } while (0)

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void alloc_shard(rmpc_handle& h, Shard& sh) {
  CK(cudaSetDevice(sh.device));
  CK(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sh.stream2, cudaStreamNonBlocking));
  cudaDeviceGetAttribute(&sh.sms, cudaDevAttrMultiProcessorCount, sh.device);
  for (auto& e : sh.ev) CK(cudaEventCreate(&e));
  const size_t n = std::max(sh.count, 1);
  const size_t zn = n * h.NT * RMPC_NV;
  CK(cudaMalloc(&sh.d_states, n * sizeof(rmpc_state)));
  CK(cudaMalloc(&sh.d_cmds, n * sizeof(rmpc_command)));
  CK(cudaMalloc(&sh.d_gaits, n * sizeof(rmpc_gait)));
  CK(cudaMalloc(&sh.d_prev, n * sizeof(rmpc_solution)));
  CK(cudaMalloc(&sh.d_prev_z, zn * sizeof(float)));
  CK(cudaMalloc(&sh.d_out, n * sizeof(rmpc_solution)));
  CK(cudaMalloc(&sh.d_z, zn * sizeof(float)));
  CK(cudaMalloc(&sh.d_soa, n * RMPC_SOA_FIELDS * sizeof(float)));
  CK(cudaMalloc(&sh.d_prof, 2 * RMPC_NUM_STAGES * sizeof(unsigned long long)));
  cudaDeviceGetAttribute(&sh.clock_khz, cudaDevAttrClockRate, sh.device);
  sh.stage_in_bytes = n * (sizeof(rmpc_state) + sizeof(rmpc_command) + sizeof(rmpc_gait) + sizeof(rmpc_solution)) +
                      zn * sizeof(float) + 8 * 256;  // 256-byte aligned sub-buffers
  sh.stage_out_bytes = n * sizeof(rmpc_solution) + zn * sizeof(float) + 2 * 256;
  CK(cudaMallocHost(&sh.h_stage_in, sh.stage_in_bytes));
  CK(cudaMallocHost(&sh.h_stage_out, sh.stage_out_bytes));
  // schedule-shared solves: a hash table of >= 2n slots and up to kSchedCap distinct
  // schedules in the store
  for (RmpcSchedBuffers& sb : sh.sched) {
    sb.agents = (int)n;
    sb.slots = 64;
    while (sb.slots < 2 * (int)n) sb.slots *= 2;
    sb.cap = (int)std::min<size_t>(n, kSchedCap);
    CK(cudaMalloc(&sb.table, (size_t)sb.slots * sizeof(unsigned long long)));
    CK(cudaMalloc(&sb.slot_id, (size_t)sb.slots * sizeof(int32_t)));
    CK(cudaMalloc(&sb.slot_of, n * sizeof(int32_t)));
    CK(cudaMalloc(&sb.pos, n * sizeof(int32_t)));
    CK(cudaMalloc(&sb.order, n * sizeof(int32_t)));
    CK(cudaMalloc(&sb.ulist, n * sizeof(int32_t)));
    CK(cudaMalloc(&sb.rep_list, (size_t)sb.cap * sizeof(int32_t)));
    CK(cudaMalloc(&sb.cnt, (size_t)sb.cap * sizeof(int32_t)));
    CK(cudaMalloc(&sb.grp_first, (size_t)sb.cap * sizeof(int32_t)));
    CK(cudaMalloc(&sb.grp_cta, ((size_t)sb.cap + 1) * sizeof(int32_t)));
    CK(cudaMalloc(&sb.n_sched, sizeof(int32_t)));
    CK(cudaMalloc(&sb.n_unshared, sizeof(int32_t)));
    CK(cudaMalloc(&sb.store, (size_t)sb.cap * rmpc_dev::store_layout(h.NT).total * sizeof(float)));
    CK(cudaMalloc(&sb.con, 4 * sizeof(double)));
    CK(cudaHostAlloc(&sb.h_nsched, sizeof(int32_t), cudaHostAllocDefault));
    {
      cudaEvent_t en = nullptr;
      CK(cudaEventCreateWithFlags(&en, cudaEventDisableTiming));
      sb.ev_nsched = en;
    }
    sb.sqpack = nullptr;
    if (rmpc_dev::sq_supported(h.NT) || rmpc_dev::sq4_supported(h.NT))
      CK(cudaMalloc(&sb.sqpack, (size_t)sb.cap * rmpc_dev::sq_layout(h.NT).priv * sizeof(float)));
    cudaStream_t side = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    sb.side = side;
    sb.ev_fork = e0;
    sb.ev_join = e1;
  }
  const int rc = rmpc_kernel_setup(rmpc_dev::MAXT);
  if (rc != 0) {
    sh.err = RMPC_ERR_CUDA;
    sh.msg = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString((cudaError_t)rc);
  }
}

void free_shard(Shard& sh) {
  cudaSetDevice(sh.device);
  if (sh.stream) cudaStreamSynchronize(sh.stream);
  if (sh.stream2) cudaStreamSynchronize(sh.stream2);
  cudaFree(sh.d_states); cudaFree(sh.d_cmds); cudaFree(sh.d_gaits); cudaFree(sh.d_prev);
  cudaFree(sh.d_prev_z); cudaFree(sh.d_out); cudaFree(sh.d_z); cudaFree(sh.d_prof); cudaFree(sh.d_soa);
  cudaFreeHost(sh.h_stage_in); cudaFreeHost(sh.h_stage_out);
  for (RmpcSchedBuffers& sb : sh.sched) {
    for (void* p : {(void*)sb.table, (void*)sb.slot_id, (void*)sb.slot_of, (void*)sb.pos, (void*)sb.order,
                    (void*)sb.ulist, (void*)sb.rep_list, (void*)sb.cnt, (void*)sb.grp_first, (void*)sb.grp_cta,
                    (void*)sb.n_sched, (void*)sb.n_unshared, (void*)sb.store, (void*)sb.sqpack,
                    (void*)sb.con})
      cudaFree(p);
    if (sb.h_nsched) cudaFreeHost(sb.h_nsched);
    if (sb.ev_nsched) cudaEventDestroy((cudaEvent_t)sb.ev_nsched);
    if (sb.side) {
      cudaStreamSynchronize((cudaStream_t)sb.side);
      cudaStreamDestroy((cudaStream_t)sb.side);
    }
    if (sb.ev_fork) cudaEventDestroy((cudaEvent_t)sb.ev_fork);
    if (sb.ev_join) cudaEventDestroy((cudaEvent_t)sb.ev_join);
  }
  for (auto& e : sh.ev) if (e) cudaEventDestroy(e);
  if (sh.stream) cudaStreamDestroy(sh.stream);
  if (sh.stream2) cudaStreamDestroy(sh.stream2);
}

// H2D (staging pageable buffers through pinned memory), kernel, D2H, synchronize.  A shard of
// more than two waves runs as up to three chunks: the first wave of CTAs, the remaining whole
// waves (second stream), the partial last wave (behind chunk 1 on the first stream).  Chunk 1's
// inputs are small, so its kernel starts early; the later chunks' H2D overlaps chunk 1's
// kernel, chunk 1's D2H overlaps the rest, the later kernels' CTAs fill the SMs as earlier
// ones finish, and only the small tail chunk's D2H is left at the end.  Per-agent results do
// not depend on the split.
// Device address of host memory the kernel can write directly (pinned, hence mapped under UVA).
template <class T>
T* mapped(T* p) {
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, (void*)p, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return static_cast<T*>(d);
}

// SoA inputs of rmpc_solve_soa: the caller's block and its row stride (floats).
struct SoaIn {
  const float* soa;
  int64_t ld;
};

// The shard's columns [begin, begin + count) of the SoA block: one 2D H2D copy (28 rows; a
// pageable block is first gathered into the pinned staging buffer), then the unpack kernel into
// the shard's FP64 records -- on `st`, in place of the three record copies.
// With `split` (squads: the schedule pass reads only the gaits), the gait rows go first on `st`
// and the state / command rows follow on the second stream, unpacked there; sh.ev[6] marks them.
void stage_soa(Shard& sh, const SoaIn& in, cudaStream_t st, bool split = false) {
  const size_t n = sh.count, b = sh.begin;
  const float* src = in.soa + b;
  size_t pitch = (size_t)in.ld * sizeof(float);
  if (!is_pinned(in.soa)) {
    float* stg = reinterpret_cast<float*>(sh.h_stage_in);
    for (int r = 0; r < RMPC_SOA_FIELDS; ++r) std::memcpy(stg + r * n, in.soa + r * in.ld + b, n * sizeof(float));
    src = stg;
    pitch = n * sizeof(float);
  }
  auto copy_rows = [&](int r0, int nr, cudaStream_t s) {
    if (pitch == n * sizeof(float))  // contiguous rows
      CK(cudaMemcpyAsync(sh.d_soa + r0 * n, src + r0 * n, nr * n * sizeof(float), cudaMemcpyHostToDevice, s));
    else
      CK(cudaMemcpy2DAsync(sh.d_soa + r0 * n, n * sizeof(float), reinterpret_cast<const char*>(src) + r0 * pitch,
                           pitch, n * sizeof(float), nr, cudaMemcpyHostToDevice, s));
  };
  int rc = 0;
  if (!split) {
    copy_rows(0, RMPC_SOA_FIELDS, st);
    if (sh.err) return;
    rc = rmpc_launch_soa_unpack(sh.d_soa, (long long)n, (int)n, sh.d_states, sh.d_cmds, sh.d_gaits, st, 0);
  } else {
    copy_rows(RMPC_SOA_PHASE, RMPC_SOA_FIELDS - RMPC_SOA_PHASE, st);
    if (sh.err) return;
    rc = rmpc_launch_soa_unpack(sh.d_soa, (long long)n, (int)n, sh.d_states, sh.d_cmds, sh.d_gaits, st, 1);
    CK(cudaEventRecord(sh.ev[7], st));
    CK(cudaStreamWaitEvent(sh.stream2, sh.ev[7], 0));
    copy_rows(0, RMPC_SOA_PHASE, sh.stream2);
    if (sh.err) return;
    if (rc == 0)
      rc = rmpc_launch_soa_unpack(sh.d_soa, (long long)n, (int)n, sh.d_states, sh.d_cmds, sh.d_gaits, sh.stream2, 2);
    CK(cudaEventRecord(sh.ev[6], sh.stream2));
  }
  if (rc != 0) {
    sh.err = RMPC_ERR_CUDA;
    sh.msg = std::string("soa_unpack_kernel launch: ") + cudaGetErrorString((cudaError_t)rc);
  }
}

// Cold start with schedule sharing: the inputs in one H2D copy each, then the whole shared
// solve (schedule pass, grouped solve) writing its records and z* straight into the pinned
// host buffers (the caller's, or the handle's staging copy for pageable ones) over PCIe while
// it runs -- the grouped solve finishes every agent at once at the end, so there is no later
// chunk whose kernel a D2H could overlap.
void run_shard_shared(rmpc_handle& h, Shard& sh, const rmpc_state* states, const rmpc_command* cmds,
                      const rmpc_gait* gaits, rmpc_solution* out, float* z_out, const SoaIn* soa) {
  const size_t n = sh.count, b = sh.begin;
  const size_t zrow = (size_t)h.NT * RMPC_NV;
  const cudaStream_t st = sh.stream;
  struct In {
    const char* src;
    char* dst;
    size_t bytes;
  };
  std::vector<In> ins;
  if (!soa)
    ins = {{reinterpret_cast<const char*>(states + b), reinterpret_cast<char*>(sh.d_states), n * sizeof(rmpc_state)},
           {reinterpret_cast<const char*>(cmds + b), reinterpret_cast<char*>(sh.d_cmds), n * sizeof(rmpc_command)},
           {reinterpret_cast<const char*>(gaits + b), reinterpret_cast<char*>(sh.d_gaits), n * sizeof(rmpc_gait)}};
  size_t off = 0;
  for (In& c : ins) {
    if (!is_pinned(c.src)) {
      std::memcpy(sh.h_stage_in + off, c.src, c.bytes);
      c.src = sh.h_stage_in + off;
      off += (c.bytes + 255) & ~size_t(255);
    }
  }
  const bool out_pinned = is_pinned(out), z_pinned = is_pinned(z_out);
  rmpc_solution* h_out = out_pinned ? out + b : reinterpret_cast<rmpc_solution*>(sh.h_stage_out);
  float* h_z = z_out ? (z_pinned ? z_out + b * zrow
                                 : reinterpret_cast<float*>(sh.h_stage_out + ((n * sizeof(rmpc_solution) + 255) & ~size_t(255))))
                     : nullptr;
  rmpc_solution* d_out = mapped(h_out);
  float* d_z = h_z ? mapped(h_z) : nullptr;
  CK(cudaEventRecord(sh.ev[0], st));
  if (h.profile) CK(cudaMemsetAsync(sh.d_prof, 0, 2 * RMPC_NUM_STAGES * sizeof(unsigned long long), st));
  // squads: the schedule pass and the store build read only the gaits, so the states and
  // commands (3/4 of the bytes) are copied on the second stream behind them and the solve waits
  // for them only where it reads them (rmpc_launch_shared's ev_inputs)
  const int path = solve_path(h, sh.sms);
  const bool split_in = !soa && path == 2;
  void* ev_inputs = nullptr;
  if (soa) {
    stage_soa(sh, *soa, st, path == 2);
    if (sh.err) return;
    if (path == 2) ev_inputs = sh.ev[6];
  }
  if (split_in) {
    CK(cudaMemcpyAsync(ins[2].dst, ins[2].src, ins[2].bytes, cudaMemcpyHostToDevice, st));  // gaits
    CK(cudaEventRecord(sh.ev[1], st));
    CK(cudaStreamWaitEvent(sh.stream2, sh.ev[1], 0));  // behind the gaits, not beside them
    for (int k = 0; k < 2; ++k)
      CK(cudaMemcpyAsync(ins[k].dst, ins[k].src, ins[k].bytes, cudaMemcpyHostToDevice, sh.stream2));
    CK(cudaEventRecord(sh.ev[6], sh.stream2));
    ev_inputs = sh.ev[6];
  } else {
    for (const In& c : ins) CK(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(sh.ev[1], st));
  }
  rmpc_dev::KParams P = make_params(h);
  P.n_agents = (int)n;
  P.states = sh.d_states;
  P.cmds = sh.d_cmds;
  P.gaits = sh.d_gaits;
  P.prof = sh.d_prof;
  // mapped host outputs: the solve writes the device buffers and copy-out kernels move the
  // results over PCIe, the first wave's beside the second wave's solve (RmpcCopyOut)
  RmpcCopyOut co{sh.stream2, sh.ev[3], sh.ev[4], d_out, d_z, sh.sms};
  const bool copyout = d_out != nullptr && d_z != nullptr;  // (records alone: written in the solve)
  P.out = copyout ? sh.d_out : (d_out ? d_out : sh.d_out);
  P.z_out = z_out ? (copyout ? sh.d_z : (d_z ? d_z : sh.d_z)) : nullptr;
  const int rc = rmpc_launch_shared(P, sh.sched[0], st, path, copyout ? &co : nullptr, ev_inputs);
  if (rc != 0) {
    sh.err = rc == (int)cudaErrorNoKernelImageForDevice ? RMPC_ERR_NO_KERNEL : RMPC_ERR_CUDA;
    sh.msg = std::string("rti_shared_kernel launch: ") + cudaGetErrorString((cudaError_t)rc);
    cudaStreamSynchronize(st);
    return;
  }
  CK(cudaEventRecord(sh.ev[2], st));
  if (!copyout) {
    if (!d_out) CK(cudaMemcpyAsync(h_out, sh.d_out, n * sizeof(rmpc_solution), cudaMemcpyDeviceToHost, st));
    if (z_out && !d_z) CK(cudaMemcpyAsync(h_z, sh.d_z, n * zrow * sizeof(float), cudaMemcpyDeviceToHost, st));
  }
  if (h.profile) CK(cudaMemcpyAsync(sh.prof, sh.d_prof, sizeof(sh.prof), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(sh.ev[5], st));
  CK(cudaStreamSynchronize(st));
  if (!out_pinned) std::memcpy(out + b, h_out, n * sizeof(rmpc_solution));
  if (z_out && !z_pinned) std::memcpy(z_out + b * zrow, h_z, n * zrow * sizeof(float));
  float t01 = 0, t12 = 0, t25 = 0;
  cudaEventElapsedTime(&t01, sh.ev[0], sh.ev[1]);
  cudaEventElapsedTime(&t12, sh.ev[1], sh.ev[2]);  // the solve, incl. the mapped output writes
  cudaEventElapsedTime(&t25, sh.ev[2], sh.ev[5]);
  sh.h2d_ms = t01;
  sh.kernel_ms = t12;
  sh.d2h_ms = t25;
}

void run_shard(rmpc_handle& h, Shard& sh, const rmpc_state* states, const rmpc_command* cmds,
               const rmpc_gait* gaits, const rmpc_solution* prev, const float* prev_z,
               rmpc_solution* out, float* z_out, const SoaIn* soa = nullptr) {
  sh.err = 0;
  if (sh.count == 0) return;
  CK(cudaSetDevice(sh.device));
  if (solve_path(h, sh.sms) != 0) {
    run_shard_shared(h, sh, states, cmds, gaits, out, z_out, soa);
    return;
  }
  const size_t n = sh.count, b = sh.begin;
  const size_t zrow = (size_t)h.NT * RMPC_NV;
  const bool use_prev = h.settings.warm_start && prev && prev_z;
  // chunks: the first wave, the remaining whole waves, the partial last wave (its D2H is the
  // only transfer left exposed at the end)
  const size_t wave = (size_t)sh.sms * rmpc_dev::cta_shape(h.NT).agents;
  size_t cut[4] = {0, n, n, n};
  int nchunks = 1;
  if (n > 2 * wave && !h.profile) {
    const size_t tail = n % wave;
    cut[1] = wave;
    nchunks = 2;
    if (tail > 0 && n - tail > wave) {
      cut[2] = n - tail;
      nchunks = 3;
    }
  }
  const cudaStream_t ss[3] = {sh.stream, sh.stream2, sh.stream};  // the tail chunk queues behind chunk 1
  struct In {
    const char* src;
    char* dst;
    size_t elem;  // bytes per agent
  };
  std::vector<In> ins;
  if (!soa)  // (SoA: the whole shard's records are unpacked on the device ahead of chunk 0)
    ins = {{reinterpret_cast<const char*>(states + b), reinterpret_cast<char*>(sh.d_states), sizeof(rmpc_state)},
           {reinterpret_cast<const char*>(cmds + b), reinterpret_cast<char*>(sh.d_cmds), sizeof(rmpc_command)},
           {reinterpret_cast<const char*>(gaits + b), reinterpret_cast<char*>(sh.d_gaits), sizeof(rmpc_gait)}};
  if (use_prev) {
    ins.push_back({reinterpret_cast<const char*>(prev + b), reinterpret_cast<char*>(sh.d_prev), sizeof(rmpc_solution)});
    ins.push_back({reinterpret_cast<const char*>(prev_z + b * zrow), reinterpret_cast<char*>(sh.d_prev_z),
                   zrow * sizeof(float)});
  }
  size_t off = 0;
  for (In& c : ins) {
    if (!is_pinned(c.src)) {
      std::memcpy(sh.h_stage_in + off, c.src, n * c.elem);
      c.src = sh.h_stage_in + off;
      off += (n * c.elem + 255) & ~size_t(255);
    }
  }
  const bool out_pinned = is_pinned(out), z_pinned = is_pinned(z_out);
  char* out_dst = out_pinned ? reinterpret_cast<char*>(out + b) : sh.h_stage_out;
  char* z_dst = nullptr;
  if (z_out)
    z_dst = z_pinned ? reinterpret_cast<char*>(z_out + b * zrow)
                     : sh.h_stage_out + ((n * sizeof(rmpc_solution) + 255) & ~size_t(255));
  CK(cudaEventRecord(sh.ev[0], ss[0]));
  if (h.profile) CK(cudaMemsetAsync(sh.d_prof, 0, 2 * RMPC_NUM_STAGES * sizeof(unsigned long long), ss[0]));
  if (nchunks > 1) CK(cudaStreamWaitEvent(ss[1], sh.ev[0], 0));
  for (int k = 0; k < nchunks; ++k) {
    const cudaStream_t st = ss[k];
    const size_t lo = cut[k], m = cut[k + 1] - cut[k];
    if (soa && k == 0) {
      stage_soa(sh, *soa, st);
      if (sh.err) return;
    }
    for (const In& c : ins)
      CK(cudaMemcpyAsync(c.dst + lo * c.elem, c.src + lo * c.elem, m * c.elem, cudaMemcpyHostToDevice, st));
    if (k == 0) CK(cudaEventRecord(sh.ev[1], st));
    if (soa && k == 0 && nchunks > 1) CK(cudaStreamWaitEvent(ss[1], sh.ev[1], 0));  // the unpacked records
    rmpc_dev::KParams P = make_params(h);
    P.n_agents = (int)m;
    P.states = sh.d_states + lo;
    P.cmds = sh.d_cmds + lo;
    P.gaits = sh.d_gaits + lo;
    P.prev = use_prev ? sh.d_prev + lo : nullptr;
    P.prev_z = use_prev ? sh.d_prev_z + lo * zrow : nullptr;
    P.out = sh.d_out + lo;
    P.z_out = z_out ? sh.d_z + lo * zrow : nullptr;
    P.prof = sh.d_prof;
    const int rc = rmpc_launch_rti(P, st);
    if (rc != 0) {
      sh.err = rc == (int)cudaErrorNoKernelImageForDevice ? RMPC_ERR_NO_KERNEL : RMPC_ERR_CUDA;
      sh.msg = std::string("rti_kernel launch: ") + cudaGetErrorString((cudaError_t)rc);
      cudaStreamSynchronize(ss[0]);
      cudaStreamSynchronize(ss[1]);
      return;
    }
    CK(cudaEventRecord(sh.ev[2 + k], st));  // kernel k done (events 2..4)
    CK(cudaMemcpyAsync(out_dst + lo * sizeof(rmpc_solution), sh.d_out + lo, m * sizeof(rmpc_solution),
                       cudaMemcpyDeviceToHost, st));
    if (z_out)
      CK(cudaMemcpyAsync(z_dst + lo * zrow * sizeof(float), sh.d_z + lo * zrow, m * zrow * sizeof(float),
                         cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(sh.ev[5 + k], st));  // results of chunk k on the host (events 5..7)
  }
  if (h.profile)
    CK(cudaMemcpyAsync(sh.prof, sh.d_prof, sizeof(sh.prof), cudaMemcpyDeviceToHost, ss[0]));
  CK(cudaStreamSynchronize(ss[0]));
  if (nchunks > 1) CK(cudaStreamSynchronize(ss[1]));
  if (!out_pinned) std::memcpy(out + b, out_dst, n * sizeof(rmpc_solution));
  if (z_out && !z_pinned) std::memcpy(z_out + b * zrow, z_dst, n * zrow * sizeof(float));
  // exposed stage times: chunk 1's H2D, first H2D done -> last kernel done, last kernel done ->
  // last results on the host
  const int last = nchunks - 1;
  float t01 = 0, t1k = 0, tkd = 0;
  cudaEventElapsedTime(&t01, sh.ev[0], sh.ev[1]);
  for (int k = 0; k < nchunks; ++k) {
    float tk = 0;
    cudaEventElapsedTime(&tk, sh.ev[1], sh.ev[2 + k]);
    t1k = std::max(t1k, tk);
  }
  cudaEventElapsedTime(&tkd, sh.ev[2 + last], sh.ev[5 + last]);
  sh.h2d_ms = t01;
  sh.kernel_ms = t1k;
  sh.d2h_ms = tkd;
}

void fill_timing(rmpc_handle& h, double total_ms) {
  rmpc_timing& t = h.timing;
  std::memset(&t, 0, sizeof(t));
  t.batch_size = h.n;
  t.devices = (int)h.shards.size();
  t.total_ms = total_ms;
  double sum[RMPC_NUM_STAGES] = {0}, sq[RMPC_NUM_STAGES] = {0};
  int clock_khz = 0;
  for (const Shard& sh : h.shards) {
    t.h2d_ms = std::max(t.h2d_ms, sh.h2d_ms);
    t.kernel_ms = std::max(t.kernel_ms, sh.kernel_ms);
    t.d2h_ms = std::max(t.d2h_ms, sh.d2h_ms);
    for (int s = 0; s < RMPC_NUM_STAGES; ++s) {
      sum[s] += (double)sh.prof[s];
      sq[s] += (double)sh.prof[RMPC_NUM_STAGES + s];
    }
    clock_khz = std::max(clock_khz, sh.clock_khz);
  }
  if (h.profile) {
    // split of the kernel time by stage (cycles summed over agents), and the per-agent stage
    // time statistics of TimingReport::mean_ms / std_ms (batch.cpp:67-77) from the SM clock
    double tot = 0;
    for (int s = 0; s < RMPC_NUM_STAGES; ++s) tot += sum[s];
    const double n = (double)h.n, cyc_ms = clock_khz > 0 ? 1.0 / clock_khz : 0.0;
    for (int s = 0; s < RMPC_NUM_STAGES; ++s) {
      if (tot > 0) t.stage_ms[s] = t.kernel_ms * sum[s] / tot;
      const double mean = sum[s] / n;
      t.stage_mean_ms[s] = mean * cyc_ms;
      t.stage_std_ms[s] = std::sqrt(std::max(0.0, sq[s] / n - mean * mean)) * cyc_ms;
    }
  }
}

// One launch of the fused kernel for `n` device-resident agents of shard `sh` on `stream`
// (NULL = the legacy default stream, as every other device entry point of the library).
int32_t launch_device(rmpc_handle& h, Shard& sh, int n, const rmpc_state* d_states, const rmpc_command* d_cmds,
                      const rmpc_gait* d_gaits, const rmpc_solution* d_prev, const float* d_prev_z,
                      rmpc_solution* d_out, float* d_z, uint8_t* d_active, void* stream) {
  if (cudaSetDevice(sh.device) != cudaSuccess) {
    cudaGetLastError();
    h.err = "cudaSetDevice failed";
    return RMPC_ERR_CUDA;
  }
  rmpc_dev::KParams P = make_params(h);
  P.n_agents = n;
  P.states = d_states;
  P.cmds = d_cmds;
  P.gaits = d_gaits;
  const bool use_prev = h.settings.warm_start && d_prev && d_prev_z && !d_active;
  P.prev = use_prev ? d_prev : nullptr;
  P.prev_z = use_prev ? d_prev_z : nullptr;
  P.out = d_out;
  P.z_out = d_z;
  P.act_out = d_active;
  P.prof = sh.d_prof;
  P.profile = 0;
  if (d_active) P.warm_start = 0;
  const int path = solve_path(h, sh.sms, d_active != nullptr);  // (the active-set solve is cold)
  const int rc = path != 0 ? rmpc_launch_shared(P, sh.sched[0], stream, path)  // cold start, shared
                           : rmpc_launch_rti(P, stream);
  if (rc != 0) {
    h.err = std::string("rti_kernel launch: ") + cudaGetErrorString((cudaError_t)rc);
    return rc == (int)cudaErrorNoKernelImageForDevice ? RMPC_ERR_NO_KERNEL : RMPC_ERR_CUDA;
  }
  return RMPC_OK;
}

}  // namespace

// FMA throughput probe (FP32 for the solve, FP64 for the PPO batch): 8 independent FMA chains
// per thread, enough resident warps to saturate every SM.  The roofline denominators
// ("of measured").
template <typename F>
__global__ void fma_peak_kernel(F* out, int iters, F a, F b) {
  F x0 = threadIdx.x * F(1e-7), x1 = x0 + F(1e-7), x2 = x0 + F(2e-7), x3 = x0 + F(3e-7);
  F x4 = x0 + F(4e-7), x5 = x0 + F(5e-7), x6 = x0 + F(6e-7), x7 = x0 + F(7e-7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const F r = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (r == F(1.2345)) out[0] = r;  // keep the chains alive
}

template <typename F>
int32_t fma_peak(int32_t device, double* tflops) {
  if (!tflops) return RMPC_ERR_INVALID_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return RMPC_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  F* d = nullptr;
  cudaMalloc(&d, sizeof(F));
  const int threads = 256, blocks = sms * 8, iters = sizeof(F) == 4 ? 4096 : 1024;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_peak_kernel<F><<<blocks, threads>>>(d, 64, F(0.999), F(1e-6));  // warm-up
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_peak_kernel<F><<<blocks, threads>>>(d, iters, F(0.999), F(1e-6));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const cudaError_t e = cudaGetLastError();
  *tflops = best;
  return e == cudaSuccess ? RMPC_OK : RMPC_ERR_CUDA;
}

extern "C" {

void rmpc_model_default(rmpc_model* p) {
  std::memset(p, 0, sizeof(*p));
  p->torso_mass = 10.0; p->torso_len = 0.4; p->torso_inertia = 10.0 * 0.4 * 0.4 / 12.0;
  p->thigh_mass = 2.5; p->thigh_len = 0.4; p->thigh_inertia = 2.5 * 0.4 * 0.4 / 12.0;
  p->shank_mass = 1.5; p->shank_len = 0.4; p->shank_inertia = 1.5 * 0.4 * 0.4 / 12.0;
  p->foot_mass = 0.5; p->foot_half_len = 0.09; p->foot_inertia = 0.5 * 0.18 * 0.18 / 12.0;
  p->ankle_drop = 0.05;
  const double lo[6] = {-1.5, 0.05, -1.2, -1.5, 0.05, -1.2}, hi[6] = {1.5, 2.4, 1.2, 1.5, 2.4, 1.2};
  const double tl[6] = {60.0, 60.0, 30.0, 60.0, 60.0, 30.0};
  for (int j = 0; j < 6; ++j) {
    p->joint_lo[j] = lo[j]; p->joint_hi[j] = hi[j]; p->qd_limit[j] = 20.0;
    p->tau_limit[j] = tl[j]; p->kp[j] = 30.0; p->kd[j] = 1.0;
  }
  p->mu = 0.8; p->gravity = 9.81; p->nominal_stagger = 0.15; p->nominal_drop = 0.75;
}

void rmpc_settings_default(rmpc_settings* s, int32_t horizon) {
  std::memset(s, 0, sizeof(*s));
  s->horizon = horizon;
  for (int i = 0; i < RMPC_MAX_HORIZON; ++i) s->dt_schedule[i] = i < horizon ? 0.05 : 0.0;
  const double wq[9] = {0.0, 500.0, 300.0, 5.0, 5.0, 5.0, 5.0, 5.0, 5.0};
  const double wqd[9] = {100.0, 100.0, 50.0, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1};
  for (int k = 0; k < 9; ++k) { s->w_q[k] = wq[k]; s->w_qd[k] = wqd[k]; }
  for (int k = 0; k < 8; ++k) s->w_f[k] = 1e-3;
  s->gait_period = 0.8; s->phase_switch = 0.5;
  s->phase_offsets[0] = 0.5; s->phase_offsets[1] = 0.5; s->phase_offsets[2] = 0.0; s->phase_offsets[3] = 0.0;
  s->z_swing = 0.075; s->v_to = 0.2; s->v_td = -0.3;
  s->n_qp = 25; s->mu = 0.6; s->sigma = 1e-6; s->rho = 0.1; s->over_relax = 1.6;
  s->warm_start = 0; s->ruiz_iters = 10;
}

void rmpc_nominal_pose(const rmpc_model* model, double q_out[RMPC_NQ]) { nominal_pose_host(*model, q_out); }

int32_t rmpc_create(const rmpc_model* model, const rmpc_settings* settings, int32_t n_agents,
                    const int32_t* devices, int32_t n_devices, rmpc_handle** out) {
  if (!out || !model || !settings) { g_create_error = "rmpc_create: NULL argument"; return RMPC_ERR_INVALID_ARG; }
  *out = nullptr;
  if (n_agents < 1) { g_create_error = "BatchRunner: n_envs must be >= 1"; return RMPC_ERR_STRUCTURAL; }
  if (settings->horizon < 2) { g_create_error = "MpcController: horizon must be >= 2"; return RMPC_ERR_STRUCTURAL; }
  if (settings->horizon > RMPC_MAX_HORIZON) { g_create_error = "MpcController: horizon > RMPC_MAX_HORIZON"; return RMPC_ERR_STRUCTURAL; }
  if (settings->n_qp < 1) { g_create_error = "AdmmSolver: n_iters must be >= 1"; return RMPC_ERR_STRUCTURAL; }
  // The reference's MPC always equilibrates (MpcSettings::admm() leaves AdmmSettings::ruiz_iters at
  // 10, mpc.hpp:49-56); the FP32 reduced system H = P^ + sigma I + rho A^T A squares the row
  // scales of an unequilibrated A and loses the 1e-4 bar without at least one Ruiz pass.
  if (settings->ruiz_iters < 1) {
    g_create_error = "rmpc_create: ruiz_iters must be >= 1 (the FP32 reduced ADMM system needs equilibration)";
    return RMPC_ERR_STRUCTURAL;
  }
  for (int i = 0; i < settings->horizon; ++i)
    if (!(settings->dt_schedule[i] > 0.0)) { g_create_error = "MpcController: dt_schedule entries must be > 0"; return RMPC_ERR_STRUCTURAL; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_create_error = "rmpc_create: no CUDA device";
    return RMPC_ERR_CUDA;
  }
  std::vector<int> devs;
  if (devices && n_devices > 0) devs.assign(devices, devices + n_devices);
  else devs.push_back(0);
  for (int d : devs)
    if (d < 0 || d >= ndev) { g_create_error = "rmpc_create: device index out of range"; return RMPC_ERR_INVALID_ARG; }
  rmpc_handle* h = new rmpc_handle();
  h->model = *model;
  h->settings = *settings;
  h->n = n_agents;
  h->NT = settings->horizon;
  nominal_pose_host(*model, h->nominal);
  std::memset(&h->timing, 0, sizeof(h->timing));
  const int G = (int)devs.size();
  h->shards.resize(G);
  for (int g = 0; g < G; ++g) {  // contiguous ranges [g n / G, (g+1) n / G)
    Shard& sh = h->shards[g];
    sh.device = devs[g];
    rmpc_shard_range(n_agents, G, g, &sh.begin, &sh.count);
    alloc_shard(*h, sh);
    if (sh.err) {
      g_create_error = sh.msg;
      for (int k = 0; k <= g; ++k) free_shard(h->shards[k]);
      delete h;
      return RMPC_ERR_CUDA;
    }
  }
  if (G > 1) h->pool.reset(new ShardPool(G - 1));
  *out = h;
  return RMPC_OK;
}

void rmpc_destroy(rmpc_handle* h) {
  if (!h) return;
  h->pool.reset();
  for (Shard& sh : h->shards) free_shard(sh);
  delete h;
}

int32_t rmpc_solve(rmpc_handle* h, const rmpc_state* states, const rmpc_command* cmds, const rmpc_gait* gaits,
                   const rmpc_solution* prev, const float* prev_z_star, rmpc_solution* out, float* z_star_out) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  if (!states || !cmds || !gaits || !out) {
    h->err = "BatchRunner::solve: input lengths != n_envs (NULL array)";
    return RMPC_ERR_STRUCTURAL;
  }
  const auto t0 = std::chrono::steady_clock::now();
  if (h->shards.size() == 1) {
    run_shard(*h, h->shards[0], states, cmds, gaits, prev, prev_z_star, out, z_star_out);
  } else {
    const std::function<void(int)> job = [&](int g) {
      run_shard(*h, h->shards[g], states, cmds, gaits, prev, prev_z_star, out, z_star_out);
    };
    h->pool->run(job);
  }
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  for (const Shard& sh : h->shards)
    if (sh.err) { h->err = sh.msg; return sh.err; }
  fill_timing(*h, ms);
  return RMPC_OK;
}

int32_t rmpc_solve_soa(rmpc_handle* h, const float* soa, int64_t ld, const rmpc_solution* prev,
                       const float* prev_z_star, rmpc_solution* out, float* z_star_out) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  if (!soa || !out) {
    h->err = "rmpc_solve_soa: NULL array";
    return RMPC_ERR_STRUCTURAL;
  }
  if (ld < h->n) {
    h->err = "rmpc_solve_soa: row stride ld < n_envs";
    return RMPC_ERR_STRUCTURAL;
  }
  const SoaIn in{soa, ld};
  const auto t0 = std::chrono::steady_clock::now();
  if (h->shards.size() == 1) {
    run_shard(*h, h->shards[0], nullptr, nullptr, nullptr, prev, prev_z_star, out, z_star_out, &in);
  } else {
    const std::function<void(int)> job = [&](int g) {
      run_shard(*h, h->shards[g], nullptr, nullptr, nullptr, prev, prev_z_star, out, z_star_out, &in);
    };
    h->pool->run(job);
  }
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  for (const Shard& sh : h->shards)
    if (sh.err) { h->err = sh.msg; return sh.err; }
  fill_timing(*h, ms);
  return RMPC_OK;
}

int32_t rmpc_solve_soa_device(rmpc_handle* h, const float* d_soa, int64_t ld, const rmpc_solution* d_prev,
                              const float* d_prev_z_star, rmpc_solution* d_out, float* d_z_star_out, void* stream) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  if (h->shards.size() != 1) {
    h->err = "rmpc_solve_soa_device: single-device handles only (rmpc_solve_soa shards host blocks)";
    return RMPC_ERR_INVALID_ARG;
  }
  if (!d_soa || !d_out) { h->err = "rmpc_solve_soa_device: NULL array"; return RMPC_ERR_STRUCTURAL; }
  if (ld < h->n) { h->err = "rmpc_solve_soa_device: row stride ld < n_envs"; return RMPC_ERR_STRUCTURAL; }
  Shard& sh = h->shards[0];
  if (cudaSetDevice(sh.device) != cudaSuccess) {
    cudaGetLastError();
    h->err = "cudaSetDevice failed";
    return RMPC_ERR_CUDA;
  }
  const int rc = rmpc_launch_soa_unpack(d_soa, (long long)ld, h->n, sh.d_states, sh.d_cmds, sh.d_gaits, stream);
  if (rc != 0) {
    h->err = std::string("soa_unpack_kernel launch: ") + cudaGetErrorString((cudaError_t)rc);
    return RMPC_ERR_CUDA;
  }
  return launch_device(*h, sh, h->n, sh.d_states, sh.d_cmds, sh.d_gaits, d_prev, d_prev_z_star, d_out, d_z_star_out,
                       nullptr, stream);
}

int32_t rmpc_solve_device(rmpc_handle* h, const rmpc_state* d_states, const rmpc_command* d_cmds,
                          const rmpc_gait* d_gaits, const rmpc_solution* d_prev, const float* d_prev_z_star,
                          rmpc_solution* d_out, float* d_z_star_out, void* stream) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  if (h->shards.size() != 1) {
    h->err = "rmpc_solve_device: multi-device handle, use rmpc_solve_device_sharded";
    return RMPC_ERR_INVALID_ARG;
  }
  if (!d_states || !d_cmds || !d_gaits || !d_out) { h->err = "rmpc_solve_device: NULL array"; return RMPC_ERR_STRUCTURAL; }
  return launch_device(*h, h->shards[0], h->n, d_states, d_cmds, d_gaits, d_prev, d_prev_z_star, d_out, d_z_star_out,
                       nullptr, stream);
}

int32_t rmpc_solve_device_sharded(rmpc_handle* h, const rmpc_state* const* d_states, const rmpc_command* const* d_cmds,
                                  const rmpc_gait* const* d_gaits, const rmpc_solution* const* d_prev,
                                  const float* const* d_prev_z_star, rmpc_solution* const* d_out,
                                  float* const* d_z_star_out, void* const* streams) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  if (!d_states || !d_cmds || !d_gaits || !d_out) { h->err = "rmpc_solve_device_sharded: NULL array"; return RMPC_ERR_STRUCTURAL; }
  for (size_t g = 0; g < h->shards.size(); ++g) {
    Shard& sh = h->shards[g];
    if (sh.count == 0) continue;
    if (!d_states[g] || !d_cmds[g] || !d_gaits[g] || !d_out[g]) {
      h->err = "rmpc_solve_device_sharded: NULL array for shard " + std::to_string(g);
      return RMPC_ERR_STRUCTURAL;
    }
    const int rc = launch_device(*h, sh, sh.count, d_states[g], d_cmds[g], d_gaits[g], d_prev ? d_prev[g] : nullptr,
                                 d_prev_z_star ? d_prev_z_star[g] : nullptr, d_out[g],
                                 d_z_star_out ? d_z_star_out[g] : nullptr, nullptr, streams ? streams[g] : nullptr);
    if (rc != RMPC_OK) return rc;
  }
  return RMPC_OK;
}

int32_t rmpc_shard_range(int32_t n_agents, int32_t n_shards, int32_t shard, int32_t* begin, int32_t* count) {
  if (n_agents < 0 || n_shards < 1 || shard < 0 || shard >= n_shards) return RMPC_ERR_INVALID_ARG;
  const int32_t b = (int32_t)((long long)shard * n_agents / n_shards);
  const int32_t e = (int32_t)((long long)(shard + 1) * n_agents / n_shards);
  if (begin) *begin = b;
  if (count) *count = e - b;
  return RMPC_OK;
}

int32_t rmpc_shard_info(const rmpc_handle* h, int32_t shard, int32_t* device, int32_t* begin, int32_t* count) {
  if (!h || shard < 0 || shard >= (int32_t)h->shards.size()) return RMPC_ERR_INVALID_ARG;
  const Shard& sh = h->shards[shard];
  if (device) *device = sh.device;
  if (begin) *begin = sh.begin;
  if (count) *count = sh.count;
  return RMPC_OK;
}

int32_t rmpc_solve_device_active_set(rmpc_handle* h, const rmpc_state* d_states, const rmpc_command* d_cmds,
                                     const rmpc_gait* d_gaits, rmpc_solution* d_out, uint8_t* d_active,
                                     void* stream) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  if (h->shards.size() != 1) { h->err = "rmpc_solve_device_active_set: single-device handles only"; return RMPC_ERR_INVALID_ARG; }
  if (!d_states || !d_cmds || !d_gaits || !d_out || !d_active) { h->err = "rmpc_solve_device_active_set: NULL array"; return RMPC_ERR_STRUCTURAL; }
  return launch_device(*h, h->shards[0], h->n, d_states, d_cmds, d_gaits, nullptr, nullptr, d_out, nullptr, d_active,
                       stream);
}

int32_t rmpc_size(const rmpc_handle* h) { return h ? h->n : 0; }
int32_t rmpc_workers(const rmpc_handle* h) { return h ? (int32_t)h->shards.size() : 0; }
int32_t rmpc_horizon(const rmpc_handle* h) { return h ? h->NT : 0; }

int32_t rmpc_last_timing(const rmpc_handle* h, rmpc_timing* out) {
  if (!h || !out) return RMPC_ERR_INVALID_ARG;
  *out = h->timing;
  return RMPC_OK;
}

const char* rmpc_last_error(const rmpc_handle* h) { return h ? h->err.c_str() : g_create_error.c_str(); }

const char* rmpc_status_message(int32_t status) {
  switch (status) {
    case RMPC_STATUS_OK: return "ok";
    case RMPC_STATUS_NONFINITE_INPUT: return "build_qp: non-finite linearization point";
    case RMPC_STATUS_DIVERGED: return "admm: non-finite iterate";
    case RMPC_STATUS_SINGULAR: return "factorization: non-positive pivot";
    default: return "unknown status";
  }
}

const char* rmpc_stage_name(int32_t stage) {
  static const char* names[RMPC_NUM_STAGES] = {"init_guess", "param", "kkt_build", "ruiz",
                                               "factorize", "admm_iters", "rnea"};
  return (stage >= 0 && stage < RMPC_NUM_STAGES) ? names[stage] : "unknown";
}

int32_t rmpc_mpc_torque(const rmpc_model* model, const rmpc_solution* sol, const rmpc_state* state,
                        double tau_out[RMPC_NJ]) {
  if (!model || !sol || !state || !tau_out) return RMPC_ERR_INVALID_ARG;
  if (sol->status != RMPC_STATUS_OK) return RMPC_ERR_STRUCTURAL;  // mpc.cpp:341-342
  for (int j = 0; j < RMPC_NJ; ++j) {  // robot.cpp:235-241
    const double t = model->kp[j] * ((double)sol->q_set[j] - state->q[3 + j]) +
                     model->kd[j] * ((double)sol->qd_set[j] - state->qd[3 + j]) + (double)sol->tau_ff[j];
    tau_out[j] = std::min(std::max(t, -model->tau_limit[j]), model->tau_limit[j]);
  }
  return RMPC_OK;
}

int32_t rmpc_set_schedule_sharing(rmpc_handle* h, int32_t enabled) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  h->share = enabled < 0 ? 0 : (enabled > 3 ? 3 : enabled);
  return RMPC_OK;
}

int32_t rmpc_set_stage_profiling(rmpc_handle* h, int32_t enabled) {
  if (!h) return RMPC_ERR_INVALID_ARG;
  h->profile = enabled ? 1 : 0;
  return RMPC_OK;
}

const char* rmpc_build_info(void) {
  return "rmpc_b200 sm_100a fused warp-pair-per-agent RTI kernel (reduced SPD block-tridiagonal ADMM, factor in TMEM, FP32 + FP64 linearization)";
}

int32_t rmpc_fma_peak(int32_t device, double* tflops) { return fma_peak<float>(device, tflops); }

int32_t rmpc_fma_peak_f64(int32_t device, double* tflops) { return fma_peak<double>(device, tflops); }

int32_t rmpc_smem_bytes(int32_t horizon) {
  if (horizon < 1 || horizon > rmpc_dev::MAXT) return -1;
  return rmpc_dev::cta_shape(horizon).smem_bytes / rmpc_dev::cta_shape(horizon).agents;
}
int32_t rmpc_agents_per_cta(int32_t horizon) {
  if (horizon < 1 || horizon > rmpc_dev::MAXT) return -1;
  return rmpc_dev::cta_shape(horizon).agents;
}
int32_t rmpc_sizeof(int32_t which) {
  switch (which) {
    case 0: return (int32_t)sizeof(rmpc_model);
    case 1: return (int32_t)sizeof(rmpc_settings);
    case 2: return (int32_t)sizeof(rmpc_state);
    case 3: return (int32_t)sizeof(rmpc_command);
    case 4: return (int32_t)sizeof(rmpc_gait);
    case 5: return (int32_t)sizeof(rmpc_solution);
    case 6: return (int32_t)sizeof(rmpc_timing);
    default: return -1;
  }
}

}  // extern "C"
