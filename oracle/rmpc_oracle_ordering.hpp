// rmpc_oracle_ordering.hpp — TEST INFRASTRUCTURE ONLY (see rmpc_oracle.hpp).
// The fill-reducing ordering that stands in for Eigen's AMDOrdering (ldl.cpp:14-35), shared by
// the oracle's LDL^T and by the Eigen shim (eigen_shim/Eigen/OrderingMethods) that the
// unmodified reference sources are compiled against in oracle/_ref.
#pragma once

#include <algorithm>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- ordering (replaces AMD)
// Approximate minimum degree (Amestoy, Davis & Duff 1996) on the quotient graph of the
// symmetric pattern of an upper-stored matrix: pivots become elements, elements adjacent to
// the pivot are absorbed, external degrees are bounded with the |L_e \ L_p| trick, elements
// with L_e inside L_p are absorbed aggressively.  No supervariable detection or dense-row
// postponement (neither matters at these sizes).  Eigen's AMDOrdering (ldl.cpp:14-35) is the
// same algorithm family; permutations may differ, which changes only rounding.
// Returns perm with old = perm[new] (the elimination order), as ldl.cpp:24-31.
inline std::vector<int> min_degree_ordering(int n, const std::vector<int>& colptr,
                                            const std::vector<int>& rowidx) {
  // Per-thread list workspace reused across calls (capacity kept; contents cleared), the
  // analogue of AMD's single workspace allocation.
  struct Lists {
    std::vector<std::vector<int>> vars, elems, members;
    std::vector<int> Lp;
  };
  thread_local Lists tls;
  Lists& ws = tls;  // one TLS lookup; the loops below use plain references
  auto& vars = ws.vars;
  auto& elems = ws.elems;
  auto& members = ws.members;
  auto& Lp = ws.Lp;
  if ((int)vars.size() < n) { vars.resize(n); elems.resize(n); members.resize(n); }
  for (int i = 0; i < n; ++i) { vars[i].clear(); elems[i].clear(); members[i].clear(); }
  for (int j = 0; j < n; ++j)
    for (int p = colptr[j]; p < colptr[j + 1]; ++p) {
      const int i = rowidx[p];
      if (i != j) { vars[i].push_back(j); vars[j].push_back(i); }
    }
  enum : char { kVar = 0, kElem = 1, kDead = 2 };
  std::vector<char> kind(n, kVar);
  std::vector<int> deg(n), head(n + 1, -1), nxt(n, -1), prv(n, -1);
  std::vector<int> mark(n, -1), wstamp(n, -1), w(n, 0);
  for (int i = 0; i < n; ++i) {  // drop duplicate neighbours
    auto& v = vars[i];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    deg[i] = (int)v.size();
  }
  auto bucket_insert = [&](int i) {
    const int d = deg[i];
    prv[i] = -1;
    nxt[i] = head[d];
    if (head[d] >= 0) prv[head[d]] = i;
    head[d] = i;
  };
  auto bucket_remove = [&](int i) {
    if (prv[i] >= 0) nxt[prv[i]] = nxt[i]; else head[deg[i]] = nxt[i];
    if (nxt[i] >= 0) prv[nxt[i]] = prv[i];
  };
  for (int i = n - 1; i >= 0; --i) bucket_insert(i);
  std::vector<int> perm;
  perm.reserve(n);
  int mindeg = 0;
  for (int k = 0; k < n; ++k) {
    while (head[mindeg] < 0) ++mindeg;
    const int p = head[mindeg];
    bucket_remove(p);
    perm.push_back(p);
    kind[p] = kElem;
    // L_p = (A_p U union of L_e, e in E_p) \ {p}; elements of E_p are absorbed into p.
    Lp.clear();
    mark[p] = k;
    for (int v : vars[p])
      if (kind[v] == kVar && mark[v] != k) { mark[v] = k; Lp.push_back(v); }
    for (int e : elems[p]) {
      if (kind[e] != kElem || e == p) continue;
      for (int v : members[e])
        if (kind[v] == kVar && mark[v] != k) { mark[v] = k; Lp.push_back(v); }
      kind[e] = kDead;
      members[e].clear();
    }
    vars[p].clear();
    elems[p].clear();
    members[p].assign(Lp.begin(), Lp.end());
    // w(e) = |L_e \ L_p| for every element adjacent to L_p.
    for (int i : Lp)
      for (int e : elems[i]) {
        if (kind[e] != kElem || e == p) continue;
        if (wstamp[e] != k) { wstamp[e] = k; w[e] = (int)members[e].size(); }
        --w[e];
      }
    const int lp_ext = (int)Lp.size() - 1;
    for (int i : Lp) {
      bucket_remove(i);
      int ext = 0;
      size_t ne = 0;
      for (int e : elems[i]) {  // prune absorbed elements; aggressive absorption when w(e)=0
        if (kind[e] != kElem || e == p) continue;
        if (wstamp[e] == k && w[e] == 0) { kind[e] = kDead; members[e].clear(); continue; }
        elems[i][ne++] = e;
        ext += (wstamp[e] == k) ? w[e] : (int)members[e].size() - 1;
      }
      elems[i].resize(ne);
      elems[i].push_back(p);
      size_t nv = 0;
      for (int v : vars[i])  // variables now reached through element p are dropped
        if (kind[v] == kVar && mark[v] != k && v != i) vars[i][nv++] = v;
      vars[i].resize(nv);
      ext += (int)nv + lp_ext;
      int d = std::min(deg[i] + lp_ext, n - k - 1);
      d = std::min(d, ext);
      deg[i] = std::max(d, 0);
      bucket_insert(i);
      if (deg[i] < mindeg) mindeg = deg[i];
    }
  }
  return perm;
}

}  // namespace oracle
