// sched_sim.c — discrete-time model of the engine's bulk schedule (dev tool).
//
// Models one solve: a stepper that publishes a source block every tau us and
// needs target block J's bulk sums ~0.35 tau before it starts block J; bulk
// agents (16 warps per SM, n_sm SMs) that process Toeplitz chunks (J, I) in
// ascending I per work unit.  An SM with k busy warps runs chunks at g(k) of
// its full rate (the measured lone-chain calibration in
// profiles/r01_bulk_variants.txt), shared evenly by its busy warps.
//
// policy 0: whole-target units, round-robin ownership J = L + a + i A (the
//           round-1 engine), EDF per agent, re-select when src_done moves.
// policy 1: units (J, s) = target J x source segment s of S blocks, dealt
//           round-robin in (J, s) order; the last unit of a target pays a
//           fixed-order reduction of its partials.
// policy 2: like 1, but segments split every target in `nseg` equal parts
//           at fixed block boundaries (S = ceil((nb - L) / nseg)).
//
// build: gcc -O2 -o tools/sched_sim tools/sched_sim.c -lm
// usage: tools/sched_sim N policy S [tau_ns_per_step] [warps_per_sm]
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define L 4
#define B 128

static double gk(int k, int wps) {  // SM rate fraction with k busy warps
  static const double x[] = {0, 1, 2, 4, 8, 16};
  static const double y[] = {0, 0.156, 0.310, 0.616, 0.887, 1.0};
  if (k <= 0) return 0;
  double kk = k * 16.0 / wps;  // a wps-warp SM at k busy behaves like 16-warp at k*16/wps? keep simple
  if (wps == 16) kk = k;
  for (int i = 1; i < 6; ++i)
    if (kk <= x[i]) return y[i - 1] + (y[i] - y[i - 1]) * (kk - x[i - 1]) / (x[i] - x[i - 1]);
  return 1.0;
}

typedef struct {
  int J, s, lo, hi;  // sources [lo, hi)
  int next;          // next source block
  int done, held;
} Unit;

int main(int argc, char** argv) {
  long long N = argc > 1 ? atoll(argv[1]) : 1000000;
  int policy = argc > 2 ? atoi(argv[2]) : 0;
  int S = argc > 3 ? atoi(argv[3]) : 0;
  double tau_step = argc > 4 ? atof(argv[4]) : 142.0;  // ns per step, stepper alone
  int wps = argc > 5 ? atoi(argv[5]) : 16;
  const int n_sm = 147;
  const double chunk_sm_us = 98304.0 / (1.74e13 / 148.0) * 1e6;  // one chunk at a full SM
  const double tau = tau_step * B / 1000.0;                       // us per block
  const int nb = (int)((N + B - 1) / B);
  const int nt = nb - L;
  const int A = n_sm * wps;
  const double red_us_per_partial = 0.15;  // fixed-order reduction: 6 KB per partial, one warp
  const double switch_cost = 0.05;         // spill/reload, in chunk units

  // ---- units
  int nseg_max = 1;
  if (policy == 2) S = (nt + S - 1) / S;
  if ((policy >= 3) && S <= 0) S = 1 << 30;  // argv S = number of segments
  if (policy >= 1 && S <= 0) S = 1 << 30;
  const int S2 = argc > 7 ? atoi(argv[7]) : S;
  const int isplit = argc > 8 ? (int)(atof(argv[8]) * nb) : nb;
  int nu = 0;
  for (int J = L; J < nb; ++J) nu += policy == 0 ? 1 : (J - L + 1 + S - 1) / S + (J - L + 1 > isplit ? (J - L + 1 - isplit) / S2 + 2 : 0);
  Unit* U = calloc(nu, sizeof(Unit));
  int* tgt_first = calloc(nb + 1, sizeof(int));
  int* tgt_left = calloc(nb + 1, sizeof(int));
  int u = 0;
  for (int J = L; J < nb; ++J) {
    tgt_first[J] = u;
    int n = J - L + 1;
    if (policy == 0) {
      U[u++] = (Unit){J, 0, 0, n, 0, 0, 0};
      tgt_left[J] = 1;
    } else {
      int k = 0;
      for (int lo = 0; lo < n; ++k) {
        int step = lo >= isplit ? S2 : S;
        int hi = lo + step;
        if (lo < isplit && hi > isplit) hi = isplit;
        if (hi > n) hi = n;
        U[u++] = (Unit){J, k, lo, hi, lo, 0, 0};
        lo = hi;
      }
      tgt_left[J] = k;
      if (k > nseg_max) nseg_max = k;
    }
  }
  // ---- ownership: unit list dealt round-robin; agent a lives on SM a % n_sm
  int* own_cnt = calloc(A, sizeof(int));
  int** own = malloc(A * sizeof(int*));
  if (policy < 4) {
    for (int i = 0; i < nu; ++i) own_cnt[i % A]++;
    for (int a = 0; a < A; ++a) own[a] = malloc((own_cnt[a] + 1) * sizeof(int)), own_cnt[a] = 0;
    for (int i = 0; i < nu; ++i) own[i % A][own_cnt[i % A]++] = i;  // ascending (J, s) per agent
  } else if (policy == 5) {
    for (int J = L; J < nb; ++J) own_cnt[(J - L) % A]++;
    for (int a = 0; a < A; ++a) own[a] = malloc((own_cnt[a] + 1) * sizeof(int)), own_cnt[a] = 0;
    for (int J = L; J < nb; ++J) { int a = (J - L) % A; own[a][own_cnt[a]++] = J; }
  } else {
    for (int J = L; J < nb; ++J) own_cnt[(J - L) % A]++;
    for (int a = 0; a < A; ++a) own[a] = malloc((own_cnt[a] + 1) * sizeof(int)), own_cnt[a] = 0;
    for (int J = L; J < nb; ++J) { int a = (J - L) % A; own[a][own_cnt[a]++] = tgt_first[J] + tgt_left[J] - 1; }
  }
  int ncol = (nb + S - 1) / S + 1;
  int* col_next = malloc(ncol * sizeof(int));
  for (int c = 0; c < ncol; ++c) col_next[c] = (c + 1) * S + L;
  int* dyn = malloc(A * sizeof(int));
  for (int a = 0; a < A; ++a) dyn[a] = -1;
  int* cur = malloc(A * sizeof(int));
  double* rem = calloc(A, sizeof(double));
  int* seen = calloc(A, sizeof(int));
  int* idle = calloc(A, sizeof(int));
  int* first_pending = calloc(A, sizeof(int));
  for (int a = 0; a < A; ++a) cur[a] = -1;
  double* ready = malloc((nb + 1) * sizeof(double));
  for (int J = 0; J <= nb; ++J) ready[J] = J < L ? 0 : -1;
  int gfirst = 0, stall = 0;
  const int sticky = getenv("SIM_STICKY") ? atoi(getenv("SIM_STICKY")) : 0;
  const int fin_first = getenv("SIM_FINFIRST") ? 1 : 0;
  double dt = argc > 6 ? atof(argv[6]) : 0.5, t = 0;
  double pos = 0;  // stepper position in steps
  double wait = 0;
  int src_done = 0;
  long long chunks = 0;
  double busy_warp_us = 0;
  int* kbusy = calloc(n_sm, sizeof(int));
  double util[64] = {0}, eff[64] = {0}, cnt[64] = {0};
  while (pos < N) {
    // stepper: advance unless the next needed block is not ready
    int Jn = (int)((pos + 0.35 * B) / B);  // block whose bulk is needed at this position
    if (Jn < nb && Jn >= L && ready[Jn] < 0) {
      wait += dt;
      if (++stall > 20000) {
        printf("STUCK t=%.1f Jn=%d src_done=%d\n", t, Jn, src_done);
        for (int k = tgt_first[Jn]; k < (Jn + 1 < nb ? tgt_first[Jn + 1] : nu); ++k)
          printf("  unit s=%d lo=%d hi=%d next=%d done=%d held=%d\n", U[k].s, U[k].lo, U[k].hi, U[k].next, U[k].done, U[k].held);
        int a = (Jn - L) % A; printf("  owner %d cur=%d dyn=%d idle=%d seen=%d rem=%f fp=%d\n", a, cur[a], dyn[a], idle[a], seen[a], rem[a], first_pending[a]);
        exit(1);
      }
    } else {
      pos += dt * 1000.0 / tau_step;
      stall = 0;
    }
    int sd = (int)(pos / B);
    if (sd > nb) sd = nb;
    if (pos >= N) sd = nb;
    src_done = sd;
    // agents: select
    memset(kbusy, 0, n_sm * sizeof(int));
    for (int a = 0; a < A; ++a) {
      if (cur[a] >= 0 && rem[a] > 0) { kbusy[a % n_sm]++; continue; }
      if (idle[a] && seen[a] == src_done) continue;  // idle, nothing new published
      // pick: continue current unit if it has work and src_done unchanged
      int pick = -1;
      if (cur[a] >= 0 && (seen[a] == src_done || sticky)) {
        Unit* x = &U[cur[a]];
        int lim = x->hi < src_done ? x->hi : src_done;
        if (!x->done && x->next < lim) pick = cur[a];
      }
      if (pick < 0 && policy == 5) {
        // owned targets: earliest J with a unit I hold (with work) or an unclaimed frontier unit
        int po = -1;
        for (int i = first_pending[a]; i < own_cnt[a] && po < 0; ++i) {
          int J = own[a][i];
          if (tgt_left[J] == 0) { if (i == first_pending[a]) first_pending[a]++; continue; }
          int n = J - L + 1;
          int nsg = (n + S - 1) / S;
          for (int k = 0; k < nsg; ++k) {
            Unit* x = &U[tgt_first[J] + k];
            if (x->lo >= src_done) break;
            if (x->done) continue;
            int lim = x->hi < src_done ? x->hi : src_done;
            if (x->next >= lim) continue;
            if (x->held == a + 1 || x->held == 0) { po = tgt_first[J] + k; break; }
          }
        }
        int pd = dyn[a];
        int jd = pd >= 0 ? U[pd].J : 1 << 30;
        int sd2 = -1;
        if (pd < 0) {
          for (int c = 0; c < ncol; ++c) {
            if (src_done < (c + 1) * S) break;
            while (col_next[c] < nb && (U[tgt_first[col_next[c]] + c].held || U[tgt_first[col_next[c]] + c].done)) col_next[c]++;
            if (col_next[c] < nb && col_next[c] < jd) { jd = col_next[c]; sd2 = c; }
          }
        }
        if (po >= 0 && (U[po].J <= jd || fin_first)) pick = po;
        else if (pd >= 0) pick = pd;
        else if (sd2 >= 0) { pick = tgt_first[jd] + sd2; dyn[a] = pick; col_next[sd2]++; }
        else pick = po;
        if (pick >= 0) U[pick].held = a + 1;
      }
      if (pick < 0 && policy == 4) {
        // A: earliest owned final segment with work
        int pa = -1;
        for (int i = first_pending[a]; i < own_cnt[a]; ++i) {
          Unit* x = &U[own[a][i]];
          if (x->done) { if (i == first_pending[a]) first_pending[a]++; continue; }
          int lim = x->hi < src_done ? x->hi : src_done;
          if (x->next < lim) { pa = own[a][i]; break; }
        }
        int pb = dyn[a];
        int jb = pb >= 0 ? U[pb].J : 1 << 30;
        int sb = -1;
        if (pb < 0) {
          for (int c = 0; c < ncol; ++c) {
            if (src_done < (c + 1) * S) break;
            if (col_next[c] < nb && col_next[c] < jb) { jb = col_next[c]; sb = c; }
          }
        }
        if (pa >= 0 && (U[pa].J <= jb || fin_first)) pick = pa;
        else if (pb >= 0) pick = pb;
        else if (sb >= 0) { pick = tgt_first[jb] + sb; dyn[a] = pick; col_next[sb]++; }
        else pick = pa;
      }
      if (pick < 0 && policy == 3) {
        if (cur[a] >= 0) U[cur[a]].held = 0;  // release (accumulators parked in the unit's slot)
        while (gfirst < nu && U[gfirst].done) ++gfirst;
        for (int i = gfirst; i < nu; ++i) {
          Unit* x = &U[i];
          if (x->done || x->held) continue;
          int lim = x->hi < src_done ? x->hi : src_done;
          if (x->next < lim) { pick = i; x->held = 1; break; }
          if (x->lo >= src_done && x->s == 0) break;  // later targets have nothing published either
        }
      }
      if (pick < 0 && policy <= 2) {
        for (int i = first_pending[a]; i < own_cnt[a]; ++i) {
          Unit* x = &U[own[a][i]];
          if (x->done) { if (i == first_pending[a]) first_pending[a]++; continue; }
          int lim = x->hi < src_done ? x->hi : src_done;
          if (x->next < lim) { pick = own[a][i]; break; }
        }
      }
      seen[a] = src_done;
      idle[a] = pick < 0;
      if (pick < 0) { cur[a] = pick; continue; }
      double c = 1.0;
      if (pick != cur[a] && U[pick].next > U[pick].lo) c += switch_cost;
      if (U[pick].next + 1 == U[pick].hi && U[pick].hi == U[pick].J - L + 1) c += 14.0 / 32.0;  // closing sweep
      if (U[pick].next + 1 == U[pick].hi && tgt_left[U[pick].J] == 1 && policy > 0)
        c += red_us_per_partial * (U[pick].s + 1) / chunk_sm_us / 16.0;
      cur[a] = pick;
      rem[a] = c;
      kbusy[a % n_sm]++;
    }
    // progress
    for (int a = 0; a < A; ++a) {
      if (cur[a] < 0 || rem[a] <= 0) continue;
      int k = kbusy[a % n_sm];
      double r = gk(k, wps) / k / chunk_sm_us * (wps == 16 ? 1.0 : 1.0);
      rem[a] -= dt * r;
      busy_warp_us += dt;
      if (rem[a] <= 0) {
        Unit* x = &U[cur[a]];
        x->next++;
        chunks++;
        if (x->next == x->hi) {
          x->done = 1;
          x->held = 0;
          if (dyn[a] == cur[a]) dyn[a] = -1;
          cur[a] = -1;
          if (--tgt_left[x->J] == 0) ready[x->J] = t;
        }
      }
    }
    {
      int tot = 0;
      for (int q = 0; q < n_sm; ++q) tot += kbusy[q];
      int bin = (int)(t / 10000.0);  // 10 ms bins
      if (bin < 64) { util[bin] += (double)tot / A; eff[bin] += 0; cnt[bin] += 1; }
      double e = 0;
      for (int q = 0; q < n_sm; ++q) e += gk(kbusy[q], wps);
      if (bin < 64) eff[bin] += e / n_sm;
      if (getenv("SIM_TRACE") && t >= atof(getenv("SIM_TRACE")) && fmod(t, 500.0) < dt) {
        int avail = 0, held = 0; long long backlog = 0;
        for (int i = gfirst; i < nu; ++i) { Unit* x = &U[i]; if (x->done) continue; int lim = x->hi < src_done ? x->hi : src_done; if (x->next < lim) { backlog += lim - x->next; if (x->held) held++; else avail++; } }
        printf("    t=%.1f stepper block %d/%d src_done %d busy %d avail-units %d held %d backlog chunks %lld wait %.2f\n", t/1000, (int)(pos / B), nb, src_done, tot, avail, held, backlog, wait/1000);
      }
    }
    t += dt;
  }
  for (int b = 0; b < 64 && cnt[b] > 0; ++b) printf("  t=%3d ms: busy warps %.3f  SM rate %.3f\n", b * 10, util[b] / cnt[b], eff[b] / cnt[b]);
  printf("N=%lld policy=%d S=%d units=%d nseg_max=%d tau=%.1fns/step: solve %.2f ms, stepper wait %.2f ms, chunks %lld, "
         "ideal bulk %.2f ms\n",
         N, policy, S, nu, nseg_max, tau_step, t / 1000, wait / 1000, chunks,
         (double)chunks * chunk_sm_us / n_sm / 1000);
  return 0;
}
