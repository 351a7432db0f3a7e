/* Research prototype (CPU): speculative levelized replay with FIFO
 * verification and order correction. Not product code.
 *
 * Given a DFG and a speculated per-device dispatch order pi, the schedule
 * is the max-plus longest path over DFG edges + queue-order edges, with
 * event "moments" (t, sub-round j) so zero-duration rounds are exact. The
 * order is then checked against the FIFO rule of replay.cpp:74-90; on a
 * mismatch the per-device FIFO order induced by the computed ready moments
 * replaces pi and the pass repeats.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

typedef uint64_t mom_t; /* t << 16 | j */
#define MJ 16



static const int64_t* g_key;
static const uint32_t* g_topo;
static const uint32_t* g_tie;
static int cmp_idx_by_key(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  int64_t kx = g_key[x], ky = g_key[y];
  if (kx != ky) return kx < ky ? -1 : 1;
  if (g_tie[x] != g_tie[y]) return g_tie[x] < g_tie[y] ? -1 : 1;
  x = g_topo[x]; y = g_topo[y];
  return x < y ? -1 : (x > y);
}
static const mom_t* g_mom;
static int cmp_idx_by_mom(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  mom_t kx = g_mom[x], ky = g_mom[y];
  if (kx != ky) return kx < ky ? -1 : 1;
  return x < y ? -1 : (x > y);
}

/* returns: >=1 iterations used on success, 0 = not converged in max_iter,
 * -1 cycle in exec graph at the last iteration, -2 unsupported */
int lev_solve(uint32_t n, const int64_t* dur, const uint32_t* dev, const uint8_t* flags,
              uint32_t D, const uint32_t* so, const uint32_t* su, const int64_t* est,
              const uint32_t* topo, const uint32_t* tie, int max_iter, int64_t* start, int64_t* end, int32_t* stats) {
  uint32_t e = so[n];
  uint32_t* indeg = calloc(n, 4);
  for (uint32_t k = 0; k < e; ++k) indeg[su[k]]++;
  for (uint32_t i = 0; i < n; ++i)
    if ((flags[i] & 1) && indeg[i] == 0) {
      free(indeg);
      return -2;
    }
  /* pi: ops per device sorted by (est, idx) */
  uint32_t* doff = calloc(D + 1, 4);
  for (uint32_t i = 0; i < n; ++i)
    if (!(flags[i] & 1)) doff[dev[i] + 1]++;
  for (uint32_t d = 0; d < D; ++d) doff[d + 1] += doff[d];
  uint32_t* pi = malloc(4 * (size_t)(doff[D] + 1));
  uint32_t* fill = malloc(4 * (size_t)(D + 1));
  memcpy(fill, doff, 4 * D);
  for (uint32_t i = 0; i < n; ++i)
    if (!(flags[i] & 1)) pi[fill[dev[i]]++] = i;
  g_key = est;
  g_topo = topo;
  g_tie = tie;
  for (uint32_t d = 0; d < D; ++d) qsort(pi + doff[d], doff[d + 1] - doff[d], 4, cmp_idx_by_key);
  uint32_t* nxt = malloc(4 * (size_t)n);   /* queue successor, or UINT32_MAX */
  uint8_t* hasprev = malloc(n);
  mom_t* R = malloc(8 * (size_t)n);  /* ready moment */
  mom_t* C = malloc(8 * (size_t)n);  /* completion moment */
  mom_t* Dm = malloc(8 * (size_t)n); /* dispatch moment */
  mom_t* Fm = malloc(8 * (size_t)n); /* free moment after op (for queue succ) */
  uint32_t* cnt = malloc(4 * (size_t)n);
  uint32_t* stack = malloc(4 * (size_t)n);
  uint32_t* qprev = malloc(4 * (size_t)n);
  int it, result = 0;
  int32_t viol_total = 0;
  for (it = 1; it <= max_iter; ++it) {
    for (uint32_t i = 0; i < n; ++i) {
      nxt[i] = UINT32_MAX;
      hasprev[i] = 0;
      qprev[i] = UINT32_MAX;
      R[i] = 0;
    }
    for (uint32_t d = 0; d < D; ++d)
      for (uint32_t k = doff[d]; k + 1 < doff[d + 1]; ++k) {
        nxt[pi[k]] = pi[k + 1];
        hasprev[pi[k + 1]] = 1;
        qprev[pi[k + 1]] = pi[k];
      }
    uint32_t top = 0;
    for (uint32_t i = 0; i < n; ++i) {
      cnt[i] = indeg[i] + hasprev[i];
      if (cnt[i] == 0) stack[top++] = i;
    }
    uint32_t done = 0;
    /* Kahn order: R[i] accumulates max over DFG preds' C */
    while (top) {
      uint32_t i = stack[--top];
      ++done;
      mom_t Ci;
      if (flags[i] & 1) {
        Dm[i] = R[i];
        Ci = R[i];
        start[i] = end[i] = (int64_t)(R[i] >> MJ);
      } else {
        mom_t F = qprev[i] == UINT32_MAX ? 0 : Fm[qprev[i]];
        mom_t M = R[i] > F ? R[i] : F;
        Dm[i] = M;
        int64_t t = (int64_t)(M >> MJ);
        start[i] = t;
        end[i] = t + dur[i];
        if (dur[i] > 0) {
          Ci = (mom_t)(t + dur[i]) << MJ;
          Fm[i] = Ci;
        } else {
          Ci = M + 1;
          Fm[i] = M;
        }
      }
      C[i] = Ci;
      for (uint32_t k = so[i]; k < so[i + 1]; ++k) {
        uint32_t s = su[k];
        if (R[s] < Ci) R[s] = Ci;
        if (--cnt[s] == 0) stack[top++] = s;
      }
      if (!(flags[i] & 1) && nxt[i] != UINT32_MAX) {
        if (--cnt[nxt[i]] == 0) stack[top++] = nxt[i];
      }
    }
    if (done != n) {
      result = -1;
      /* cycle: rebuild pi by FIFO over partial info is undefined; stop */
      break;
    }
    /* verify + build sigma */
    int32_t viol = 0;
    for (uint32_t d = 0; d < D; ++d) {
      uint32_t a = doff[d], b = doff[d + 1];
      for (uint32_t k = a; k < b; ++k) {
        uint32_t q = pi[k];
        int64_t Tq = (int64_t)(R[q] >> MJ);
        for (uint32_t j = k + 1; j < b; ++j) {
          uint32_t y = pi[j];
          int64_t Ty = (int64_t)(R[y] >> MJ);
          if (Ty < Tq) { viol++; if (getenv("LEVDBG") && viol < 6) fprintf(stderr, "it%d dev %u k=%u q=%u R=%llu/%llu D=%llu/%llu dur=%lld | y=%u R=%llu/%llu (T dip) j-k=%u\n", it, d, k-a, q, R[q]>>MJ, R[q]&0xffff, Dm[q]>>MJ, Dm[q]&0xffff, (long long)dur[q], y, R[y]>>MJ, R[y]&0xffff, j-k); goto next_dev; }
          if (Ty > Tq) break;
          if (R[y] <= Dm[q] && y < q) { viol++; if (getenv("LEVDBG") && viol < 6) fprintf(stderr, "it%d dev %u q=%u R=%llu/%llu D=%llu/%llu | y=%u R=%llu/%llu (idx)\n", it, d, q, R[q]>>MJ, R[q]&0xffff, Dm[q]>>MJ, Dm[q]&0xffff, y, R[y]>>MJ, R[y]&0xffff); goto next_dev; }
        }
      }
    next_dev:;
    }
    viol_total += viol; if (getenv("LEVIT")) fprintf(stderr, "[%d:%d]", it, viol);
    if (viol == 0) {
      result = it;
      break;
    }
    /* sigma: per device FIFO simulation on the computed ready moments, with
     * the causality rule: y is eligible only once every op x of the device
     * with D_old(x) < R(y) has been placed (pi is sorted by D_old). */
    g_mom = R;
    for (uint32_t d = 0; d < D; ++d) {
      uint32_t a = doff[d], b = doff[d + 1];
      uint32_t m = b - a;
      if (!m) continue;
      uint32_t* old = malloc(4 * m);
      memcpy(old, pi + a, 4 * m);
      uint32_t* arr = malloc(4 * m);
      memcpy(arr, pi + a, 4 * m);
      qsort(arr, m, 4, cmp_idx_by_mom);
      uint32_t* need = malloc(4 * m);   /* per arr entry */
      uint32_t* posof = malloc(4 * m);  /* arr entry -> position in old */
      uint8_t* popped = calloc(m, 1);
      for (uint32_t z = 0; z < m; ++z) {
        mom_t r = R[arr[z]];
        uint32_t lo = 0, hi = m;  /* first position with Dm >= r */
        while (lo < hi) { uint32_t md = (lo + hi) / 2; if (Dm[old[md]] < r) lo = md + 1; else hi = md; }
        need[z] = lo;
      }
      for (uint32_t w = 0; w < m; ++w) cnt[old[w]] = w; /* cnt reused as op -> old pos */
      for (uint32_t z = 0; z < m; ++z) posof[z] = cnt[arr[z]];
      uint32_t* pend = malloc(4 * m);
      uint32_t np_ = 0, nx = 0, outk = a, fp = 0;
      mom_t F = 0;
      while (outk < b) {
        if (np_ == 0 && nx < m && R[arr[nx]] > F) F = R[arr[nx]];
        while (nx < m && R[arr[nx]] <= F) pend[np_++] = nx++;
        uint32_t bi = UINT32_MAX;
        for (uint32_t z = 0; z < np_; ++z) {
          uint32_t ez = pend[z];
          if (need[ez] > fp) continue;
          if (bi == UINT32_MAX) { bi = z; continue; }
          uint32_t x = arr[ez], y = arr[pend[bi]];
          int64_t tx = (int64_t)(R[x] >> MJ), ty = (int64_t)(R[y] >> MJ);
          if (tx < ty || (tx == ty && x < y)) bi = z;
        }
        if (bi == UINT32_MAX) { fprintf(stderr, "no eligible!\n"); abort(); }
        uint32_t ez = pend[bi];
        pend[bi] = pend[--np_];
        uint32_t q = arr[ez];
        popped[posof[ez]] = 1;
        while (fp < m && popped[fp]) ++fp;
        pi[outk++] = q;
        int64_t t = (int64_t)(F >> MJ);
        if (dur[q] > 0) F = (mom_t)(t + dur[q]) << MJ;
      }
      free(pend); free(arr); free(old); free(need); free(posof); free(popped);
    }
  }
  if (it > max_iter) result = 0;
  if (stats) stats[0] = viol_total;
  free(indeg); free(doff); free(pi); free(fill); free(nxt); free(hasprev);
  free(R); free(C); free(Dm); free(Fm); free(cnt); free(stack); free(qprev);
  return result;
}

/* est for ops with known[i]==0: max over preds of est end, in Kahn order */
void lev_est(uint32_t n, const int64_t* dur, const uint8_t* flags, const uint32_t* so,
             const uint32_t* su, const uint8_t* known, int64_t* est, uint32_t* topo) {
  uint32_t pos = 0;
  uint32_t* cnt = calloc(n, 4);
  int64_t* rdy = calloc(n, 8);
  uint32_t* st = malloc(4 * (size_t)n);
  for (uint32_t k = 0; k < so[n]; ++k) cnt[su[k]]++;
  uint32_t top = 0;
  for (uint32_t i = 0; i < n; ++i) if (!cnt[i]) st[top++] = i;
  while (top) {
    uint32_t i = st[--top];
    if (!known[i] || est[i] < rdy[i]) est[i] = rdy[i];
    topo[i] = pos++;
    int64_t en = est[i] + ((flags[i] & 1) ? 0 : dur[i]);
    for (uint32_t k = so[i]; k < so[i + 1]; ++k) {
      uint32_t s = su[k];
      if (rdy[s] < en) rdy[s] = en;
      if (--cnt[s] == 0) st[top++] = s;
    }
  }
  free(cnt); free(rdy); free(st);
}
