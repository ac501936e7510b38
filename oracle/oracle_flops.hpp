// oracle_flops.hpp — TEST INFRASTRUCTURE ONLY (see rmpc_oracle.hpp).
// Counted<double>: an FP64 scalar whose arithmetic increments per-stage operation counters.
// Instantiating the oracle with it counts the reference algorithm's floating-point work per
// agent-solve exactly (the roofline's FLOP_alg).
#pragma once

#include <cmath>
#include <cstdint>

namespace oracle {

struct OpCount {
  int64_t add = 0, mul = 0, div = 0, sqrt = 0, trig = 0, cmp = 0;
  int64_t flops() const { return add + mul + div + sqrt + trig; }
};
inline thread_local OpCount g_ops[8];

struct Cd {
  double v;
  Cd() : v(0.0) {}
  Cd(double x) : v(x) {}  // NOLINT: implicit on purpose (T(1.0) etc.)
  explicit operator double() const { return v; }
};

#define ORACLE_CNT(field) (++g_ops[g_stage].field)
inline Cd operator+(Cd a, Cd b) { ORACLE_CNT(add); return Cd(a.v + b.v); }
inline Cd operator-(Cd a, Cd b) { ORACLE_CNT(add); return Cd(a.v - b.v); }
inline Cd operator*(Cd a, Cd b) { ORACLE_CNT(mul); return Cd(a.v * b.v); }
inline Cd operator/(Cd a, Cd b) { ORACLE_CNT(div); return Cd(a.v / b.v); }
inline Cd operator-(Cd a) { return Cd(-a.v); }
inline Cd& operator+=(Cd& a, Cd b) { ORACLE_CNT(add); a.v += b.v; return a; }
inline Cd& operator-=(Cd& a, Cd b) { ORACLE_CNT(add); a.v -= b.v; return a; }
inline Cd& operator*=(Cd& a, Cd b) { ORACLE_CNT(mul); a.v *= b.v; return a; }
inline Cd& operator/=(Cd& a, Cd b) { ORACLE_CNT(div); a.v /= b.v; return a; }
inline bool operator<(Cd a, Cd b) { ORACLE_CNT(cmp); return a.v < b.v; }
inline bool operator>(Cd a, Cd b) { ORACLE_CNT(cmp); return a.v > b.v; }
inline bool operator<=(Cd a, Cd b) { ORACLE_CNT(cmp); return a.v <= b.v; }
inline bool operator>=(Cd a, Cd b) { ORACLE_CNT(cmp); return a.v >= b.v; }
inline bool operator==(Cd a, Cd b) { ORACLE_CNT(cmp); return a.v == b.v; }
inline bool operator!=(Cd a, Cd b) { ORACLE_CNT(cmp); return a.v != b.v; }
inline Cd abs(Cd a) { return Cd(std::fabs(a.v)); }
inline Cd sqrt(Cd a) { ORACLE_CNT(sqrt); return Cd(std::sqrt(a.v)); }
inline Cd sin(Cd a) { ORACLE_CNT(trig); return Cd(std::sin(a.v)); }
inline Cd cos(Cd a) { ORACLE_CNT(trig); return Cd(std::cos(a.v)); }
#undef ORACLE_CNT

}  // namespace oracle
