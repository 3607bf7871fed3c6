// Simulated annealing over (sub-block slot permutation, consumer lane permutation) of the
// pull SpMV under the shared-memory bank model of tools/pull_lane_perm.py, for a given
// position of the record's pad word (before slot `gap`; 9 = at the end).
//   gcc -O2 -o /tmp/sa tools/pull_perm_anneal.c -lm && /tmp/sa <seed> <fix_slots> <gap>
// Results (2 seeds each): gap 9 (pad at the end) 34/7 = 4.86 wavefronts per 16-byte load
// (+1 split block); gap 4 4.43; gap 3 and 6: 30/7 = 4.29 (+1 split) -- the layout in
// csrc/sso_internal.h (PULL_SUB_POS, PULL_SUB_GAP = 3) and the lane table in csrc/pcg.cu.
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#define C 12
static int lanes[32];   // unit id or -1
static int slot[9]; static int gap = 9;
static int words(int u, int t, int i, int bi) {
  int j = u / 3, h = u % 3, sb = t / 2, half = t % 2;
  if (j < 5) { int q = slot[3 * sb + h]; return 80 * C + 19 * (bi + j) + 2 * q + (q >= gap) + half; }
  { int q = slot[3 * h + sb]; return 80 * i + 19 * (j - 5) + 2 * q + (q >= gap) + half; }
}
static int phases(int* w) {  // w[32], -1 inactive
  int tot = 0;
  for (int q = 0; q < 4; ++q) {
    int cnt[8] = {0}, mx = 0;
    for (int l = 8 * q; l < 8 * q + 8; ++l) if (w[l] >= 0) { int b = w[l] & 7; if (++cnt[b] > mx) mx = cnt[b]; }
    tot += mx;
  }
  return tot;
}
static double cost(void) {
  int tot = 0, w[32];
  for (int i = 0; i < C; ++i) {
    int bi = 5 * i;
    for (int t = 0; t < 6; ++t) {
      for (int l = 0; l < 32; ++l) w[l] = lanes[l] < 0 ? -1 : words(lanes[l], t, i, bi);
      tot += phases(w);
    }
    for (int l = 0; l < 32; ++l) w[l] = lanes[l] < 0 ? -1 : 27 * (i / 4) + lanes[l];
    tot += phases(w);
  }
  int split = 0;
  for (int j = 0; j < 9; ++j) {
    int qs = 0;
    for (int l = 0; l < 32; ++l) if (lanes[l] >= 0 && lanes[l] / 3 == j) qs |= 1 << (l / 8);
    split += __builtin_popcount(qs) - 1;
  }
  return (double)tot / (C * 7) + 0.25 * split;
}
int main(int argc, char** argv) {
  int seed = argc > 1 ? atoi(argv[1]) : 1;
  int fixslot = argc > 2 ? atoi(argv[2]) : 0; gap = argc > 3 ? atoi(argv[3]) : 9;
  srand(seed);
  for (int l = 0; l < 32; ++l) lanes[l] = l < 27 ? l : -1;
  for (int s = 0; s < 9; ++s) slot[s] = s;
  for (int l = 31; l > 0; --l) { int k = rand() % (l + 1); int x = lanes[l]; lanes[l] = lanes[k]; lanes[k] = x; }
  if (!fixslot) for (int s = 8; s > 0; --s) { int k = rand() % (s + 1); int x = slot[s]; slot[s] = slot[k]; slot[k] = x; }
  double c = cost(), best = c;
  int bl[32], bs[9];
  for (int l = 0; l < 32; ++l) bl[l] = lanes[l];
  for (int s = 0; s < 9; ++s) bs[s] = slot[s];
  double T = 1.0;
  for (long it = 0; it < 3000000; ++it) {
    T = 1.0 * pow(0.001, (double)it / 3000000);
    int mv = (!fixslot && rand() % 5 == 0);
    int a, b;
    if (mv) { a = rand() % 9; b = rand() % 9; int x = slot[a]; slot[a] = slot[b]; slot[b] = x; }
    else { a = rand() % 32; b = rand() % 32; int x = lanes[a]; lanes[a] = lanes[b]; lanes[b] = x; }
    double n = cost();
    if (n <= c || exp((c - n) / T) > (double)rand() / RAND_MAX) {
      c = n;
      if (c < best) { best = c; for (int l = 0; l < 32; ++l) bl[l] = lanes[l]; for (int s = 0; s < 9; ++s) bs[s] = slot[s]; }
    } else {
      if (mv) { int x = slot[a]; slot[a] = slot[b]; slot[b] = x; }
      else { int x = lanes[a]; lanes[a] = lanes[b]; lanes[b] = x; }
    }
  }
  printf("gap %d best %.4f slots", gap, best);
  for (int s = 0; s < 9; ++s) printf(" %d", bs[s]);
  printf(" lanes");
  for (int l = 0; l < 32; ++l) printf(" %d", bl[l] < 0 ? 31 : bl[l]);
  printf("\n");
  return 0;
}
