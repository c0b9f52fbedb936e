/* hull_stats.c -- hull-shape statistics of the paper's monotone CHT on histogram
 * rows, to size the hull kernel's shared rings and its eager pop tests.
 * Tooling only: not on the product path, not a test oracle.
 *
 * Input: int32 rows [E][N+1] (raw, little endian) in argv[1], N = argv[2], M = argv[3].
 * Per layer m it runs the CHT over the support rows (c_j > 0; reading R13) with the rational
 * pop rule (cross <= 0, the oracle's F6 tie rules) and reports: the largest deque, the mean deque
 * size, and per row the distributions of back / front pops; per row over all M layers (one warp
 * step of the lockstep kernel) the distribution of the MAXIMUM back / front pops.
 *
 * Build: gcc -O2 -o tools/hull_stats tools/hull_stats.c
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef long long ll;
#define MAXM 128
#define H 12

int main(int argc, char** argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: hull_stats rows.bin N M [max_entries]\n");
    return 2;
  }
  FILE* f = fopen(argv[1], "rb");
  const int N = atoi(argv[2]), M = atoi(argv[3]);
  const int maxE = argc > 4 ? atoi(argv[4]) : 1 << 30;
  int32_t* row = malloc(sizeof(int32_t) * (N + 1));
  ll* P = malloc(sizeof(ll) * (N + 1));
  int* js = malloc(sizeof(int) * (N + 1));
  ll* e_prev = malloc(sizeof(ll) * (N + 1));   /* e_{m-1} at support row index */
  ll* e_cur = malloc(sizeof(ll) * (N + 1));
  ll* qb = malloc(sizeof(ll) * (N + 2));
  int* qs = malloc(sizeof(int) * (N + 2));
  int* bp = malloc(sizeof(int) * (N + 1) * MAXM);   /* back pops [row][m] */
  int* fp = malloc(sizeof(int) * (N + 1) * MAXM);
  ll maxdq[MAXM] = {0}, sumdq[MAXM] = {0}, rows_tot = 0;
  ll over[4] = {0};   /* entries whose max deque over layers 1-16 / all exceeds 32 / 16 thresholds */
  ll hb[H] = {0}, hf[H] = {0}, hbmax[H] = {0}, hfmax[H] = {0}, steps = 0;
  int E = 0;
  while (E < maxE && fread(row, sizeof(int32_t), N + 1, f) == (size_t)(N + 1)) {
    int K = 0;
    ll acc = 0;
    P[0] = 0;
    for (int j = 1; j <= N; ++j) {
      acc += row[j];
      P[j] = acc;
      if (row[j] > 0) js[K++] = j;
    }
    for (int k = 0; k < K; ++k) e_prev[k] = 0;   /* e_0 = 0 */
    int emax_lo = 0, emax_hi = 0;   /* max deque over layers 1-32 / 33-64 for this entry */
    for (int m = 1; m <= M; ++m) {
      int fr = 0, bk = -1;
      for (int k = 0; k < K; ++k) {
        const int j = js[k];
        const ll in = k ? e_prev[k - 1] : 0;       /* e_{m-1}(j-1): value at previous support row */
        const ll nb = in + (ll)j * P[j - 1];
        int pops = 0;
        while (bk - fr >= 1) {                      /* pop back while not strictly below */
          const ll as = qs[bk - 1] - j, ab = qb[bk - 1] - nb, ks = qs[bk] - j, kb = qb[bk] - nb;
          if ((__int128)as * kb <= (__int128)ab * ks) {
            --bk;
            ++pops;
          } else {
            break;
          }
        }
        ++bk;
        qb[bk] = nb;
        qs[bk] = j;
        const ll x = P[j];
        int fpops = 0;
        while (bk > fr && qb[fr + 1] - (ll)qs[fr + 1] * x < qb[fr] - (ll)qs[fr] * x) {
          ++fr;
          ++fpops;
        }
        e_cur[k] = qb[fr] - (ll)qs[fr] * x;
        const int sz = bk - fr + 1;
        if (sz > maxdq[m - 1]) maxdq[m - 1] = sz;
        if (m <= 32 && sz > emax_lo) emax_lo = sz;
        if (m > 32 && sz > emax_hi) emax_hi = sz;
        sumdq[m - 1] += sz;
        bp[(size_t)k * MAXM + m - 1] = pops;
        fp[(size_t)k * MAXM + m - 1] = fpops;
        hb[pops < H ? pops : H - 1]++;
        hf[fpops < H ? fpops : H - 1]++;
      }
      memcpy(e_prev, e_cur, sizeof(ll) * K);
    }
    for (int k = 0; k < K; ++k) {
      int mb = 0, mf = 0;
      for (int m = 0; m < M; ++m) {
        if (bp[(size_t)k * MAXM + m] > mb) mb = bp[(size_t)k * MAXM + m];
        if (fp[(size_t)k * MAXM + m] > mf) mf = fp[(size_t)k * MAXM + m];
      }
      hbmax[mb < H ? mb : H - 1]++;
      hfmax[mf < H ? mf : H - 1]++;
      ++steps;
    }
    rows_tot += K;
    over[0] += emax_lo > 32;
    over[1] += emax_hi > 16;
    over[2] += emax_lo > 31 || emax_hi > 31;
    over[3] += emax_hi > 24;
    ++E;
  }
  printf("entries %d, N %d, M %d, support rows/entry %.1f\n", E, N, M, (double)rows_tot / E);
  printf("entries with deque > 32 in layers 1-32: %lld; > 16 in 33-64: %lld; > 31 anywhere: %lld; > 24 in 33-64: %lld\n",
         over[0], over[1], over[2], over[3]);
  printf("layer: max deque / mean deque\n");
  for (int m = 0; m < M; ++m)
    printf("  m=%2d  max %4lld  mean %6.2f\n", m + 1, maxdq[m], (double)sumdq[m] / rows_tot);
  const ll cells = rows_tot * (ll)M;
  printf("pops per (row, layer):   k: back frac | front frac\n");
  for (int h = 0; h < H; ++h)
    printf("  %2d%s  %.4f | %.4f\n", h, h == H - 1 ? "+" : " ", (double)hb[h] / cells, (double)hf[h] / cells);
  printf("max pops over the %d layers per row (one lockstep warp step): k: back | front\n", M);
  for (int h = 0; h < H; ++h)
    printf("  %2d%s  %.4f | %.4f\n", h, h == H - 1 ? "+" : " ", (double)hbmax[h] / steps, (double)hfmax[h] / steps);
  return 0;
}
