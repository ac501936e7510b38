// rmpc_device.cuh — launch parameters and shared-memory layout of the fused RTI-MPC kernel.
//
// One warp solves one agent (MpcController::rti_step, /root/reference/proj/src/mpc.cpp:248-338)
// end to end.  The ADMM linear system of the reference (quasi-definite KKT, qp.cpp:11-34, solved
// by sparse LDL^T, ldl.cpp:123-192) is replaced by its mathematically identical reduced form
//     (P^ + sigma I + rho A^T A) x~ = sigma x - q^ + A^T (rho z - y),   z~ = A^ x~,
// which is block tridiagonal over horizon nodes (26 x 26 blocks) and is solved by block
// elimination with explicit Schur-complement inverses S_i^-1 kept in tensor memory (TMEM):
// TMEM lane j holds row j of every block the warp owns, so a row is one tcgen05.ld and the
// per-agent shared memory drops to the QP data (~30 KB at T = 10, six agents per SM).
// See DESIGN.md for the derivation and the HBM / shared-memory budget.
#pragma once

#include <stdint.h>
#include <stdlib.h>

#include "../../include/rmpc_b200.h"

namespace rmpc_dev {

constexpr int NV = 26, NQ = 9, NF = 8, NC = 4, NJ = 6;
constexpr int MAXT = RMPC_MAX_HORIZON;
constexpr int SROWS = 29;     // TMEM lanes of a node block: 26 rows of S_i^-1, then W_b^T
constexpr int TCOLS = 32;     // TMEM columns per node block: S_i^-1 row j, then W_b[j] (26..28)
constexpr int MAX_AGENTS = 6; // agents (warp pairs) per CTA: 384 threads, <= 168 registers
constexpr int DENSE_AGENTS = 8;  // dense variant: 512 threads, <= 128 registers (short horizons)
constexpr int NSLOT = 40;     // constraint-row slots per node block
constexpr int NINIT = 18;     // initial-state rows
constexpr int INIT0 = 12;     // initial-state rows live in block -1, slots [12, 30)

// Row slots of node i (padded universal pattern; unused slots are zero rows with lo=hi=0,
// an exact ADMM no-op):
//   [0, 9)   integration rows of interval i      (mpc.cpp:138-148), exist for i < T-1
//   [9, 12)  base-dynamics rows of interval i     (mpc.cpp:150-175), exist for i < T-1
//   [12, 28) contact c = (s-12)/4, t = (s-12)%4   (mpc.cpp:181-218)
//              t0,t1: friction pair (stance) or zero-force rows (swing)
//              t2: stance x-velocity on qd / swing height on q (i >= 1); t3: stance z-velocity
//   [28, 34) joint position boxes, [34, 40) joint velocity boxes (mpc.cpp:220-232), i >= 1
// Block -1 (before node 0) is all-zero except the 18 initial-state rows (mpc.cpp:126-136) at
// slots [12, 30); node 0 sees it as its "previous node", so every node has the same pattern.

// Per-node coefficient block (floats).  Unscaled A values during setup/Ruiz, scaled A^ after.
constexpr int C_A1 = 0;       // [9]: integration row k on q_{i+1,k}
constexpr int C_A2 = 9;       // [9]: ... on q_{i,k}
constexpr int C_A3 = 18;      // [9]: ... on qd_{i+1,k};  [27, 36) stays zero
constexpr int C_DYNV = 36;    // [3][20]: dynamics row b on node-i vars 9..25 (index j - 9)
constexpr int C_DYNU = 96;    // [3][12]: dynamics row b on qd_{i+1,k}
constexpr int C_FORCE = 132;  // [4][4]: contact c rows t0 (Fx,Fz), t1 (Fx,Fz)
constexpr int C_JA = 148;     // [4][9]: row t2 on qd_k (stance velocity; zero for swing)
constexpr int C_JB = 184;     // [4][9]: row t3 on qd_k (stance; zero for swing)
constexpr int C_BOX = 220;    // [12]: joint q boxes (6) then qd boxes (6)
constexpr int C_INIT = 232;   // [18]: initial-state rows (node 0 only, rows in block -1)
constexpr int C_G = 250;      // [9]: G_bb' = v_b^T S_i^-1 v_b' (dynamics rows)
constexpr int C_JAQ = 260;    // [4][9]: row t2 on q_k (swing height; zero for stance)
constexpr int C_SIZE = 296;
constexpr int C_ZERO = 27;    // an entry that is always 0

// Split of the horizon for the two-sided (twisted) elimination: warp 0 owns nodes [0, m)
// eliminated top-down plus the middle node m, warp 1 owns (m, T) eliminated bottom-up.
// m = (T-1)/2 balances the two chains: even T (10): the top eliminates T/2-1 nodes plus the
// middle, the bottom T/2 (forward 5 | 5, backward 4 | 5); odd T (5): (T-1)/2 each plus the
// middle.  Both halves hold at most ceil(T/2) node blocks either way.
__host__ __device__ inline int mid_node(int NT) { return NT >= 2 ? (NT - 1) / 2 : 0; }

// Per-node vectors, V_STRIDE floats each; [26, 28) are spare (gamma of the forward sweep).
constexpr int V_X = 0;    // ADMM x (scaled space)
constexpr int V_QH = 1;   // q^ = e * q
constexpr int V_E = 2;    // Ruiz column scale e
constexpr int V_S = 3;    // r_i -> s_i -> x~_i -> next r_i
constexpr int V_NUM = 4;
constexpr int V_STRIDE = 28;
constexpr int G_SCR = 160;    // 12 x 13 G block (+ pad) of the factorization

struct KParams {
  int32_t NT, n_qp, ruiz_iters, warm_start;
  int32_t n_agents, profile;
  int32_t agents_per_cta, spill_nodes, tmem_cols;
  int32_t sq_cta_base;  // rti_squad_kernel: CTA index of this launch's first CTA (split launches)
  // Schedule pass for squads: the store is built from the nominal state (the cold-start QP
  // matrices, scales and factor depend on the schedule alone; the squads recompute every
  // agent-dependent part), so the pass reads only the gaits and the states / commands may still
  // be in flight: finiteness of the state and command is checked in the count kernel instead.
  int32_t synth_rep;
  // launch shape: full_ctas CTAs of agents_per_cta agents, then CTAs of tail_agents (the
  // last, partial wave spread over every SM at fewer agents per CTA)
  int32_t full_ctas, tail_agents;
  double dt[MAXT];
  double wq[NQ], wqd[NQ], wf[NF];
  double z_swing, v_to, v_td;
  double mu, sigma, rho, alpha;
  double m_link[7], I_link[7];
  double torso_len, thigh_len, shank_len, foot_half, ankle_drop, gravity;
  double jlo[NJ], jhi[NJ], qdlim[NJ];
  double nominal[NQ];
  double weight;  // total mass * gravity
  const rmpc_state* states;
  const rmpc_command* cmds;
  const rmpc_gait* gaits;
  const rmpc_solution* prev;
  const float* prev_z;
  rmpc_solution* out;
  float* z_out;
  uint8_t* act_out;  // optional: final active set, (T+1) x NSLOT codes per agent
  unsigned long long* prof;  // [2 RMPC_NUM_STAGES] cycle sums and sums of squares (profile only)
  // Schedule-shared factorization (cold start).  With warm_start off, the QP
  // matrices, the Ruiz scaling and the factor depend only on the contact schedule (the stance
  // flags of every node), so they are computed once per distinct schedule (mode 1, one warp
  // pair per schedule) into `store` and loaded by every agent of that schedule (mode 0).
  int32_t mode;              // 0 solve, 1 build the schedule store (no ADMM, no outputs)
  int32_t store_cap;         // schedules the store holds; ids >= cap solve unshared
  int32_t store_stride;      // floats per schedule (store_layout)
  int32_t pad2_;
  const int32_t* slot_of;    // hash slot of each agent's schedule, -1 = unshared
  const int32_t* slot_id;    // hash slot -> schedule id (-1 = over capacity)
  const int32_t* rep_list;   // mode 1: the agent that represents schedule id
  const int32_t* n_sched;    // number of schedule ids
  float* store;
  // shared-schedule solve (rti_shared_kernel): agents grouped by schedule, each CTA serves up to
  // agents_per_cta agents of one group; the rest run rti_kernel over an agent list
  const int32_t* order;      // agent indices grouped by schedule
  const int32_t* grp_cta;    // per schedule id: first CTA (prefix sum), [n_groups] = total
  const int32_t* grp_first;  // per schedule id: first position in `order`
  const int32_t* grp_count;  // per schedule id: agents
  const int32_t* agent_list; // rti_kernel: solve these agents (NULL = 0..n_agents-1)
  int32_t* n_list;           // its length (device); rti_shared_kernel appends fallbacks
  int32_t* list_out;         // = agent_list, writable (fallbacks of rti_shared_kernel)
  float* sqpack;             // per schedule id: the squad image (rti_squad_kernel, sq_pack_kernel)
  const double* con_pz;      // contact heights of the nominal pose (sched_key_kernel), [4]
};

// One schedule's entry in the store (floats, 16-byte aligned regions): the Ruiz-scaled
// coefficient blocks (incl. the G_dd entries of the factorization), the column scales e, the
// row scales d, the stance flags + factorization status, the factor's node blocks as TMEM
// rows (32 lanes x 32 columns per node) and the representative's scaled q^ (the squad solve
// replaces its four agent-dependent components).
struct StoreLayout {
  int coef, e, d, rows, flags, blocks, qh, total;
};
__host__ __device__ inline StoreLayout store_layout(int NT) {
  StoreLayout L;
  int o = 0;
  L.coef = o;   o += ((NT + 1) * C_SIZE + 3) & ~3;
  L.e = o;      o += (NT * NV + 3) & ~3;
  L.d = o;      o += ((NT + 1) * NSLOT + 3) & ~3;
  L.rows = o;   o += (NT + 1) * NSLOT * 2;       // scaled {lo, hi} of the representative
  L.flags = o;  o += (NT + 1 + 3) & ~3;  // NT flag words, then the status word (1 = factor ok)
  L.blocks = o; o += NT * 32 * TCOLS;
  L.qh = o;     o += (NT * NV + 3) & ~3;
  L.total = o;
  return L;
}

// Shared-memory footprint of one agent (warp pair) in floats, every region 16-byte aligned.
struct Layout {
  int scr, coef, vec, row, tt, dsc, bc, flags, spill, total;
};
constexpr int SPILL_BLK = 32 * TCOLS;  // a node block kept in shared memory (swizzled rows)

__host__ __device__ inline int align4(int x) { return (x + 3) & ~3; }

// spill_nodes: node blocks per warp that do not fit the warp's TMEM share (both warps of the
// agent get the same space).
__host__ __device__ inline Layout make_layout(int NT, int spill_nodes = 0) {
  Layout L;
  int o = 0;
  // scratch: Ruiz's second d, the two 12 x 13 G blocks of the factorization, z* rows (FP64)
  const int nscr = (NT + 1) * NSLOT > 2 * G_SCR ? (NT + 1) * NSLOT : 2 * G_SCR;
  L.scr = o;   o += align4(nscr);
  L.coef = o;  o += (NT + 1) * C_SIZE;              // block -1 first
  L.vec = o;   o += NT * V_NUM * V_STRIDE;
  L.row = o;   o += 4 * (NT + 1) * NSLOT;           // float4 {lo, hi, z, t = rho z - y}
  L.tt = o;    o += (NT + 1) * NSLOT;               // t of every row again, unit stride (column view)
  L.dsc = o;   o += (NT + 1) * NSLOT;               // Ruiz row scale d
  L.bc = o;    o += 128;                            // per warp: 2 x 32 broadcast buffers
  L.flags = o; o += align4(NT);
  L.spill = o; o += 2 * spill_nodes * SPILL_BLK;
  L.total = o;
  return L;
}

inline int smem_bytes(int NT, int spill_nodes = 0) { return make_layout(NT, spill_nodes).total * 4; }

// Nodes owned by one warp (top: [0, m], bottom: (m, T)), i.e. TMEM blocks per warp.
__host__ __device__ inline int nodes_per_warp(int NT) {
  const int m = mid_node(NT), a = m + 1, b = NT - 1 - m;
  return a > b ? a : b;
}

// CTA shape: A agents = 2A warps; warp w can address only TMEM lane quarter w % 4, whose 512
// columns (16 node blocks of 32) are split evenly between the warps of that quarter.  A warp's
// first `tm_nodes(quarter)` node blocks live in TMEM, the rest ("spill") in shared memory.
// Two compiled variants: the dense one (8 agents, 128 registers per thread) whenever all node
// blocks fit TMEM at 4 warps per quarter (T <= 8) and 8 agents' shared memory fits; otherwise
// the wide one, A = the largest count <= MAX_AGENTS (168 registers) whose shared memory, spill
// included, fits 227 KB.  Measured at 16 k agents: dense is 6-14% faster for T = 2..8 (more
// warps per SM outweigh the register cap); the cap costs ~10% at equal occupancy (T = 10).
__host__ __device__ inline int warps_in_quarter(int A, int q) { return (2 * A - q + 3) / 4; }
__host__ __device__ inline int tm_nodes(int NT, int A, int q) {
  const int nw = nodes_per_warp(NT), cap = 16 / warps_in_quarter(A, q);
  return nw < cap ? nw : cap;
}
struct CtaShape {
  int agents, spill_nodes, tmem_cols, smem_bytes;
  bool dense;
};
inline CtaShape cta_shape(int NT) {
  CtaShape c;
  const int nw = nodes_per_warp(NT);
  int A = MAX_AGENTS;
  c.dense = nw <= tm_nodes(NT, DENSE_AGENTS, 0) && DENSE_AGENTS * smem_bytes(NT, 0) <= 227 * 1024 - 128;
  if (c.dense) {
    A = DENSE_AGENTS;
    c.spill_nodes = 0;
  } else {
    for (;; --A) {
      c.spill_nodes = nw - tm_nodes(NT, A, 0);  // quarter 0 holds the most warps
      if (A == 1 || A * smem_bytes(NT, c.spill_nodes) <= 227 * 1024 - 128) break;
    }
  }
  c.agents = A;
  const int need = warps_in_quarter(A, 0) * tm_nodes(NT, A, 0) * TCOLS;
  int cols = 32;
  while (cols < need) cols *= 2;
  c.tmem_cols = cols;
  c.smem_bytes = A * smem_bytes(NT, c.spill_nodes);
  return c;
}

// Shared-schedule CTA (rti_shared_kernel): one schedule's coefficients, d and flags once per
// CTA, the factor once in TMEM (top-half node blocks in lane quarters 0 / 2, bottom half in
// 1 / 3, read by every warp pair of the CTA); per agent only its vectors, rows and scratch.
struct LayoutShared {
  int coef, d, flags, cta_total;   // CTA region
  int scr, vec, row, tt, bc, total;  // per agent
};
__host__ __device__ inline LayoutShared make_layout_shared(int NT) {
  LayoutShared L;
  int o = 0;
  L.coef = o;  o += (NT + 1) * C_SIZE;
  L.d = o;     o += (NT + 1) * NSLOT;
  L.flags = o; o += align4(NT);
  L.cta_total = o;
  o = 0;
  L.scr = o;   o += 256;                       // z* rows of nodes 0, 1 (FP64)
  L.vec = o;   o += NT * V_NUM * V_STRIDE;
  L.row = o;   o += 4 * (NT + 1) * NSLOT;
  L.tt = o;    o += (NT + 1) * NSLOT;
  L.bc = o;    o += 128;
  L.total = o;
  return L;
}
constexpr int SHARED_AGENTS = 8;  // rti_shared_kernel: up to 8 warp pairs (512 threads, 128 registers)
struct CtaShapeShared {
  int agents, tmem_cols, smem_bytes;
};
// Agents per shared-schedule CTA: 6 warp pairs under 168 registers (rti_shared_kernel<6>, no
// spills) or 8 under a 128-register cap (<8>, spills in the ADMM loop).  Measured at 16 384
// agents (tools/time_solve.py): 6 is faster for every horizon but T = 3 (within 2%), e.g.
// T = 10: 3.67 vs 3.93 ms, T = 20: 6.75 vs 8.17 ms.  RMPC_SHARED_AGENTS=8 selects the other
// variant (tuning experiments).
inline int shared_agents_cap(int NT) {
  (void)NT;
  static const int env = [] {
    const char* e = getenv("RMPC_SHARED_AGENTS");
    return e ? atoi(e) : 0;
  }();
  return env == SHARED_AGENTS ? SHARED_AGENTS : MAX_AGENTS;
}
inline CtaShapeShared cta_shape_shared(int NT, int cap = SHARED_AGENTS) {
  CtaShapeShared c;
  const LayoutShared L = make_layout_shared(NT);
  int A = cap;
  while (A > 1 && (L.cta_total + A * L.total) * 4 > 227 * 1024 - 256) --A;
  c.agents = A;
  int cols = 32;
  while (cols < nodes_per_warp(NT) * TCOLS) cols *= 2;
  c.tmem_cols = cols;
  c.smem_bytes = (L.cta_total + A * L.total) * 4;
  return c;
}

// ------------------------------------------------------------------------- squads
// Lane-per-agent schedule-shared solve (rmpc_squad.cuh).
constexpr int SQ_PACK_SLICES = 8;  // sq_pack_kernel CTAs per schedule
constexpr int SQ_MAXT = 10;   // horizons served by squads (5 node slabs of 96 TMEM columns per thread)
constexpr int SQ_SLAB = 98;   // TMEM columns per own node
constexpr int SQ_X = 0;       // x (26)
constexpr int SQ_S = 26;      // s / x~ (26), then gamma (3) and 3 spare (the matvec writes 32 rows)
constexpr int SQ_TI = 58;     // t of the node's interval rows, slots 0..11
constexpr int SQ_TO = 70;     // t of the node's own rows, slots 12..39
constexpr int SQ_TINIT = 490; // top thread: t of the 18 initial-state rows (block -1)
constexpr int SQ_MROW = 28;   // floats per packed matrix row (26 + 2 zero: 16-byte aligned rows)
constexpr int SQ_MF = 32 * SQ_MROW;  // packed node matrix: S^-1 rows 0..25, W_b^T rows 26..28, zero rows 29..31
constexpr int SQ_NXI = 21;    // private scratch: the backward step's xi (12 top, 21 bottom)
constexpr int SQ_NZ = 20;     // z of a node's inequality rows: t0/t1 of the 4 contacts, 12 boxes
constexpr int SQ_PRIV = 28;   // private shared elements per own node: 20 z, 4 swing lo, 4 q^ parts
// finish scratch (reuses the matrices): x_m, z* rows 0/1 (FP64), the bottom's partials, and per
// warp a 32 x 27 transpose buffer that turns lane-per-agent results into contiguous records
constexpr int SQ_FIN_XP = 26 * 32 + 2 * 2 * NV * 32 + 5 * 32;
constexpr int SQ_FIN = SQ_FIN_XP + 2 * 32 * 27;

// Shared-memory layout of one squad (floats, 16-byte aligned regions).
struct SqLayout {
  int coef, mf, lo, hi, d, e, qh, flags, priv, cross, total, priv_warp;
};
__host__ __device__ inline SqLayout sq_layout(int NT) {
  SqLayout L;
  int o = 0;
  const int nb = nodes_per_warp(NT);
  L.coef = o;  o += (NT + 1) * C_SIZE;  // block -1 first
  L.mf = o;    o += NT * SQ_MF > SQ_FIN ? NT * SQ_MF : SQ_FIN;
  L.lo = o;    o += (NT + 1) * NSLOT;   // the schedule's scaled bounds (block -1 first)
  L.hi = o;    o += (NT + 1) * NSLOT;
  L.d = o;     o += (NT + 1) * NSLOT;   // Ruiz row scales
  L.e = o;     o += align4(NT * NV);    // Ruiz column scales
  L.qh = o;    o += align4(NT * NV);    // the schedule's scaled q^
  L.flags = o; o += align4(NT + 1);     // stance bits per node, then the factorization status
  L.priv_warp = 32 * (nb * SQ_PRIV + NINIT + SQ_NXI);
  L.priv = o;  o += 2 * L.priv_warp;
  L.cross = o; o += 32 * 82;
  L.total = o;
  return L;
}
inline int sq_smem_bytes(int NT) { return 2 * sq_layout(NT).total * 4; }
inline bool sq_supported(int NT) { return NT >= 2 && NT <= SQ_MAXT && sq_smem_bytes(NT) <= 227 * 1024 - 256; }

// ------------------------------------------------------------------------- long squads
// Horizons 11..20: one squad of 32 agents per CTA on four warps (rmpc_squad4.cuh).
// Cross-thread elements of a long squad ([element][lane]); the squad ones (rmpc_squad.cuh) first.
constexpr int S4X_BAD = 56;   // first non-finite iteration of each warp (4)
constexpr int S4X_SAME = 60;  // schedule check of each warp (4)
constexpr int S4X_HTF = 64;   // top forward hand-over: g_int (9), g (3), interval nA-1 rows t (12)
constexpr int S4X_HBF = 88;   // bottom forward hand-over: g'_int (9), g' (3)
constexpr int S4X_HTB = 100;  // top backward hand-over: x~_nA (26)
constexpr int S4X_HBB = 126;  // bottom backward hand-over: x~_{i0-1} (26)
constexpr int S4X_BT = 152;   // t of interval i0-1's rows (12)
constexpr int S4X_UA = 164;   // the middle node's u from top-B (26)
constexpr int S4X_N = 190;
// named barriers of a long squad (one squad per CTA; 0 is __syncthreads)
constexpr int S4B_MID = 1, S4B_TM = 2, S4B_TF = 3, S4B_TB = 4, S4B_BF = 5, S4B_BB = 6, S4B_ALL = 7;

struct Sq4Layout {
  int img;  // the schedule image (sq_layout's region [0, priv))
  int priv, priv_warp, cross, total;
};
__host__ __device__ inline Sq4Layout sq4_layout(int NT) {
  const SqLayout L = sq_layout(NT);
  Sq4Layout S;
  S.img = 0;
  S.priv_warp = 32 * (5 * SQ_PRIV + NINIT + SQ_NXI);
  S.priv = L.priv;
  S.cross = S.priv + 4 * S.priv_warp;
  S.total = S.cross + 32 * S4X_N;
  return S;
}
// node ranges: top-A [0, nA), top-B [nA, m], bottom-B [m+1, i0), bottom-A [i0, T)
__host__ __device__ inline int sq4_na(int NT) { return (mid_node(NT) + 1) / 2; }
__host__ __device__ inline int sq4_i0(int NT) { return NT - (NT - 1 - mid_node(NT)) / 2; }
inline int sq4_smem_bytes(int NT) { return sq4_layout(NT).total * 4; }
inline bool sq4_supported(int NT) {
  if (NT <= SQ_MAXT || NT > 20) return false;
  const int m = mid_node(NT), nA = sq4_na(NT), i0 = sq4_i0(NT);
  const int w1 = nA > m + 1 - nA ? nA : m + 1 - nA, w2 = i0 - m - 1 > NT - i0 ? i0 - m - 1 : NT - i0;
  const int w = w1 > w2 ? w1 : w2;
  return w <= 5 && NT * SQ_MF >= 4 * 32 * 27 + 2 * 2 * NV * 32 + 4 * 5 * 32 + 32 &&
         sq4_smem_bytes(NT) <= 227 * 1024 - 256;
}



}  // namespace rmpc_dev

// Launch the fused kernel for params.n_agents agents on `stream` (implemented in
// rmpc_kernel.cu).  Returns a cudaError_t value.
int rmpc_launch_rti(const rmpc_dev::KParams& params, void* stream);

// Device buffers of the schedule-shared path, one set per chunk of a shard (rmpc_host.cu).
struct RmpcSchedBuffers {
  unsigned long long* table;  // open-addressing hash of schedule keys, `slots` entries
  int32_t* slot_id;           // per slot: schedule id
  int32_t* slot_of;           // per agent: slot, -1 = unshared
  int32_t* rep_list;          // per schedule id: representative agent
  int32_t* n_sched;           // schedule count
  int32_t* cnt;               // per schedule id: agents (cap)
  int32_t* pos;               // per agent: position within its group, -1 = unshared
  int32_t* grp_cta;           // cap + 1
  int32_t* grp_first;         // cap
  int32_t* order;             // agents grouped by schedule
  int32_t* ulist;             // unshared agents (and fallbacks)
  int32_t* n_unshared;
  float* store;               // cap x store_layout(T).total floats
  float* sqpack;              // cap x sq_layout(T).priv floats (squads), or NULL
  double* con;                // [4] contact heights of the nominal pose (the cold guess of every node)
  int32_t* h_nsched;          // pinned host copy of n_sched (host outputs: one or two squad waves?)
  void* ev_nsched;            // recorded after that copy (cudaEvent_t)
  int32_t slots, cap, agents;
  // the grouping pass (count, scan, scatter) runs on a side stream beside the store build:
  // fork after the key kernel, join before the group solve (cudaStream_t / cudaEvent_t)
  void* side;
  void* ev_fork;
  void* ev_join;
};
// The whole cold-start solve with schedule sharing for params.n_agents agents on `stream`:
// hash every agent's stance schedule, build the store (one factorization per schedule), group
// the agents by schedule, solve the groups (rti_shared_kernel: one schedule per CTA) and the
// rest (rti_kernel over an agent list, dispatched from the device).  Nine launches, no host
// synchronisation.
// variant 1: warp-pair-per-agent CTAs of one schedule (rti_shared_kernel, bit-identical to the
// per-agent solve); 2: lane-per-agent squads (rti_squad_kernel) where the horizon fits them.
// End-to-end outputs of a squad solve (host solve with outputs in pinned, mapped host memory):
// the solve writes params.out / params.z_out (device buffers), its squads run as two launches
// (the first wave of CTAs, then the rest), and sq_copyout_kernel moves the first wave's records
// and z* rows to h_out / h_z on stream2 while the second launch runs; the rest follows on
// `stream`.  Events ev_a / ev_b order the two copies.  Only the squad path splits; elsewhere the
// solve writes h_out / h_z directly.
struct RmpcCopyOut {
  void* stream2;
  void* ev_a;
  void* ev_b;
  rmpc_solution* h_out;  // device address of the mapped host records
  float* h_z;            // device address of the mapped host z* (NULL: no z*)
  int sms;
};
// ev_inputs (cudaEvent_t, optional): recorded when the states and commands have arrived on the
// device -- the squad pass starts on the gaits alone and waits for it only where it reads them.
int rmpc_launch_shared(const rmpc_dev::KParams& params, const RmpcSchedBuffers& b, void* stream, int variant,
                       const RmpcCopyOut* co = nullptr, void* ev_inputs = nullptr);
int rmpc_kernel_setup(int NT);  // cudaFuncSetAttribute for the dynamic shared memory
// SoA FP32 inputs (rmpc_solve_soa, RMPC_SOA_* rows of `ld` floats) -> the per-agent FP64
// records the solve kernels read; one thread per agent, coalesced row loads.
// part: 0 every row, 1 the gait rows only, 2 the state and command rows only.
int rmpc_launch_soa_unpack(const float* soa, long long ld, int n, rmpc_state* states, rmpc_command* cmds,
                           rmpc_gait* gaits, void* stream, int part = 0);
