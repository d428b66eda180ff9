// Per-frame posterior finalization shared by the dense/grouped path (align.cu) and the sparse
// (approximate + exact) path (align_grouped.cu): gmm.py:413-438.
#pragma once
#include <math.h>

#include "common.cuh"

namespace tvk {

constexpr int kMaxTopK = 32;

// Emit the kept entries of one frame sorted by component: comps[e], wts[e] (f32), returns the count.
// ll[j] are the full-covariance log-likelihoods of the selected components id[j] (selection order).
__device__ inline int finalize_frame(int K, double prune, const double* ll_in, const int* id, int* oc, float* ow) {
  double ll[kMaxTopK];
  double mx = -INFINITY;
  for (int j = 0; j < K; j++) {
    ll[j] = ll_in[j];
    mx = fmax(mx, ll[j]);
  }
  if (!isfinite(mx)) mx = 0.0;  // scipy logsumexp convention
  double s = 0.0;
  for (int j = 0; j < K; j++) s += exp(ll[j] - mx);
  const double lse = log(s) + mx;
  int nkeep = 0, best = 0;
  for (int j = 0; j < K; j++) {
    ll[j] = exp(ll[j] - lse);  // posterior over the selection
    if (ll[j] > ll[best]) best = j;
    if (ll[j] >= prune) nkeep++;
  }
  const bool degenerate = nkeep == 0;
  double tot = 0.0;
  for (int j = 0; j < K; j++) {
    const bool keep = degenerate ? (j == best) : (ll[j] >= prune);
    if (!keep) ll[j] = 0.0;
    tot += ll[j];
  }
  int n = 0;
  for (int j = 0; j < K; j++) {
    const bool keep = degenerate ? (j == best) : (ll[j] >= prune);
    if (!keep) continue;
    const float wv = (float)(ll[j] / tot);
    const int c = id[j];
    int p = n++;
    while (p > 0 && oc[p - 1] > c) {
      oc[p] = oc[p - 1];
      ow[p] = ow[p - 1];
      p--;
    }
    oc[p] = c;
    ow[p] = wv;
  }
  return n;
}

// The kept set is already known (bitmask over the selection): weights exp(ll_k - lse_kept), which
// equals post_k / sum_kept post of the reference; a single kept entry has weight 1.
__device__ inline int finalize_known(int K, unsigned kept, const double* ll_in, const int* id, int* oc, float* ow) {
  double mx = -INFINITY;
  for (int j = 0; j < K; j++)
    if ((kept >> j) & 1u) mx = fmax(mx, ll_in[j]);
  double s = 0.0;
  if (__popc(kept) > 1)
    for (int j = 0; j < K; j++)
      if ((kept >> j) & 1u) s += exp(ll_in[j] - mx);
  const double lse = __popc(kept) > 1 ? log(s) + mx : 0.0;
  int n = 0;
  for (int j = 0; j < K; j++) {
    if (!((kept >> j) & 1u)) continue;
    const float wv = __popc(kept) > 1 ? (float)exp(ll_in[j] - lse) : 1.0f;
    const int c = id[j];
    int p = n++;
    while (p > 0 && oc[p - 1] > c) {
      oc[p] = oc[p - 1];
      ow[p] = ow[p - 1];
      p--;
    }
    oc[p] = c;
    ow[p] = wv;
  }
  return n;
}

}  // namespace tvk
