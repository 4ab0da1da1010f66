// revolve.cpp -- binomial checkpoint schedule (host, integer-only).
//
// Restates checkpointing.py:32-170: the closed-form minimal recomputation
// count p~(nt, nc) (Eq. 9 of the paper), the stage-storing split recurrence
// and the action generator with its two segment shapes (a plain segment whose
// start state is positioned, and a segment whose last record is already held
// in a slot).  The action list is shared by every CTA of the reverse kernel:
// all samples follow the same fixed time grid.
#include "revolve.h"

#include <algorithm>
#include <stdexcept>
#include <unordered_map>

namespace ob {

static long long binom(long long n, long long k) {
  if (k < 0 || n < 0 || k > n) return 0;
  k = std::min(k, n - k);
  long long r = 1;
  for (long long i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

long long revolve_count(int nt, int nc) {
  if (nt < 1 || nc < 1) throw std::invalid_argument("need nt >= 1 and nc >= 1");
  if (nt == 1) return 0;
  long long t = 1;
  while (!(binom(nc + t - 1, t - 1) < nt && nt <= binom(nc + t, t))) ++t;
  return (t - 1) * nt - binom(nc + t, t - 1) + 1;
}

namespace {
struct SplitTable {
  std::unordered_map<long long, long long> memo;
  long long cost(int len, int c) {
    if (len <= 1 || c >= len - 1) return 0;
    if (c == 1) return (long long)(len - 1) * (len - 2) / 2;
    const long long key = ((long long)len << 20) | c;
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    long long best = -1;
    for (int m = 1; m < len; ++m) {
      const long long v = (m - 1) + cost(len - m, c - 1) + cost(m, c);
      if (best < 0 || v < best) best = v;
    }
    memo[key] = best;
    return best;
  }
  int split(int len, int c) {
    long long best = -1;
    int bm = 1;
    for (int m = 1; m < len; ++m) {
      const long long v = (m - 1) + cost(len - m, c - 1) + cost(m, c);
      if (best < 0 || v < best) { best = v; bm = m; }
    }
    return bm;
  }
};

struct Gen {
  SplitTable tab;
  std::vector<Action> out;
  void A(int i, int j) { out.push_back({kAdvance, -1, i, j}); }
  void S(int k) { out.push_back({kStore, k, -1, -1}); }
  void L(int k) { out.push_back({kRestore, k, -1, -1}); }
  void R(int k) { out.push_back({kReverse, k, -1, -1}); }

  void plain(int o, int n, int c, int anchor) {
    if (n == 0) return;
    const int last = o + n - 1;
    if (n == 1) { A(o, o + 1); R(o); return; }
    if (c >= n - 1) {
      for (int k = o; k < last; ++k) { A(k, k + 1); S(k); }
      A(last, last + 1);
      R(last);
      for (int k = last - 1; k >= o; --k) { L(k); R(k); }
      return;
    }
    if (c == 1) {
      A(o, o + 1); S(o); A(o + 1, o + n); R(last);
      for (int k = last - 1; k > o; --k) { L(o); A(o + 1, k + 1); R(k); }
      L(o); R(o);
      return;
    }
    const int m = tab.split(n, c);
    A(o, o + m); S(o + m - 1);
    plain(o + m, n - m, c - 1, o + m - 1);
    L(anchor);
    slotted(o, m, c, anchor);
  }

  void slotted(int o, int n, int c, int anchor) {
    const int last = o + n - 1;
    if (n == 1) { R(o); return; }
    if (c >= n - 1) {
      for (int k = o; k < last - 1; ++k) { A(k, k + 1); S(k); }
      A(last - 1, last);
      R(last); R(last - 1);
      for (int k = last - 2; k >= o; --k) { L(k); R(k); }
      return;
    }
    if (c == 1) {
      R(last);
      for (int k = last - 1; k >= o; --k) { L(anchor); A(o, k + 1); R(k); }
      return;
    }
    const int m = tab.split(n, c);
    A(o, o + m); S(o + m - 1);
    slotted(o + m, n - m, c - 1, o + m - 1);
    L(anchor);
    slotted(o, m, c, anchor);
  }
};
}  // namespace

std::vector<Action> revolve_schedule(int nt, int nc) {
  if (nt < 1 || nc < 1) throw std::invalid_argument("need nt >= 1 and nc >= 1");
  Gen g;
  g.plain(0, nt, nc, -1);
  return g.out;
}

}  // namespace ob
