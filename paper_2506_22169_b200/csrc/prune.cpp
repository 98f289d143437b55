// prune.cpp — the paper's search space for the two-GEMM chain and its pruning funnel (host only).
//
// PAPER.md §III-A/§III-C: the space is every tiling expression (24 deep permutations of m, n, k, h
// and the 2 flat expressions mn(k,h), nm(k,h)) times every tile vector whose entries are
// multiples of 16 up to the padded dimension, P:261's 109,051,904 candidates at
// M = N = 1024, K = H = 512.  The four rules of P:283-290 then cut it down (Fig. 7):
//   Rule 1  bind the spatial loops of the final output (m, h of E) to blockIdx and delete them
//           wherever they appear; expressions with the same remaining sub-tiling expression are one
//           class ("both mhnk and mnkh yield the same sub-tiling expression nk"); the first
//           expression in enumeration order represents its class;
//   Rule 2  drop a class in which the producer's reduction loop k encloses the producer's spatial
//           loop n (Fig. 6(b): `kn` caches many partial C tiles);
//   Rule 3  every axis: keep a tile that divides the dimension; a padded tile on a power-of-2
//           dimension is rejected, otherwise the padding ratio must stay < 0.05;
//   Rule 4  Eq. (1) over the in-block tiles A (TM x TK), B (TK x TN), C (TM x TN),
//           D (TN x TH), E (TM x TH), times the element size; reject when > 1.2 Shm_max.
// DESIGN.md R21 lists these readings (SPEC.md's pruner module takes the same ones).  The B200
// selector (selector.cpp) searches the kernel families that implement the surviving class `nk`
// (mh(n(k(...)))) instead of this space; mbci_prune_funnel reproduces the paper's Fig. 7 study.
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mbci.h"
#include "selector.h"

namespace mbci {

namespace {

std::vector<std::string> tiling_expressions() {
  std::vector<std::string> out;
  std::string axes = "hkmn";   // sorted, so next_permutation walks all 4! orders
  do out.push_back(axes); while (std::next_permutation(axes.begin(), axes.end()));
  out.push_back("mn(k,h)");
  out.push_back("nm(k,h)");
  return out;
}

// Rule 1 key: delete m and h; a Seq left with one child prints as n(k).
std::string sub_tiling_expression(const std::string& e) {
  std::string out;
  for (char c : e)
    if (c != 'm' && c != 'h') out.push_back(c);
  for (const char* pat : {"(,", ",)"}) {
    size_t p;
    while ((p = out.find(pat)) != std::string::npos) out.replace(p, 2, pat[0] == '(' ? "(" : ")");
  }
  size_t p;
  while ((p = out.find("()")) != std::string::npos) out.erase(p, 2);
  return out;
}

bool rule2_reject_key(const std::string& key) {
  const size_t k = key.find('k'), n = key.find('n');
  return k != std::string::npos && n != std::string::npos && k < n;
}

std::vector<int64_t> rule3_tiles(int64_t dim) {
  std::vector<int64_t> out;
  for (int64_t t = 16; t < dim + 16; t += 16)
    if (!rule3_reject(dim, t)) out.push_back(t);
  return out;
}

}  // namespace

mbci_status_t prune_funnel(int64_t M, int64_t N, int64_t K, int64_t H, int32_t elem_bytes, int64_t shm_max,
                           mbci_funnel_t* f) {
  const std::vector<std::string> exprs = tiling_expressions();
  std::vector<std::string> keys;
  for (const auto& e : exprs) {
    const std::string k = sub_tiling_expression(e);
    if (std::find(keys.begin(), keys.end(), k) == keys.end()) keys.push_back(k);
  }
  int32_t kept = 0;
  for (const auto& k : keys) kept += rule2_reject_key(k) ? 0 : 1;
  const int64_t dims[4] = {M, N, K, H};
  int64_t v_raw = 1;
  for (int64_t d : dims) v_raw *= (d + 15) / 16;
  const auto tm = rule3_tiles(M), tn = rule3_tiles(N), tk = rule3_tiles(K), th = rule3_tiles(H);
  const int64_t v3 = static_cast<int64_t>(tm.size() * tn.size() * tk.size() * th.size());
  if (v3 > (int64_t{1} << 30)) return MBCI_ERR_UNSUPPORTED;
  const double limit = 1.2 * static_cast<double>(shm_max);
  int64_t v4 = 0;
  for (int64_t a : tm)
    for (int64_t b : tn)
      for (int64_t c : tk)
        for (int64_t d : th) {
          const double shm = static_cast<double>(a * c + c * b + a * b + b * d + a * d) * elem_bytes;
          if (!(shm > limit)) ++v4;
        }
  f->expr_raw = static_cast<int32_t>(exprs.size());
  f->expr_rule1 = static_cast<int32_t>(keys.size());
  f->expr_rule2 = kept;
  f->tile_vectors = v_raw;
  f->tile_vectors_rule3 = v3;
  f->tile_vectors_rule4 = v4;
  f->raw = f->expr_raw * v_raw;
  f->after_rule1 = f->expr_rule1 * v_raw;
  f->after_rule2 = kept * v_raw;
  f->after_rule3 = kept * v3;
  f->after_rule4 = kept * v4;
  return MBCI_OK;
}

}  // namespace mbci
