// LRU simulation of 128-B line fetches for the edge-ID indirected reverse (alpha rows of 32 B).
// input: order[nrows] (schedule), rev_off[V+1], rev_eid[E]; W = rows in flight (round-robin interleave)
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
typedef struct { int64_t key; int32_t prev, next; } Node;
static int64_t *htab; static int32_t *hval; static int64_t hcap;
static int64_t hfind(int64_t k) { uint64_t h = (uint64_t)k * 0x9E3779B97F4A7C15ull; int64_t i = h & (hcap - 1);
  while (htab[i] != -1 && htab[i] != k) i = (i + 1) & (hcap - 1); return i; }
// deletion with backward-shift for linear probing
static void hdel(int64_t i) { int64_t j = i; htab[i] = -1;
  for (;;) { j = (j + 1) & (hcap - 1); if (htab[j] == -1) return;
    uint64_t h = (uint64_t)htab[j] * 0x9E3779B97F4A7C15ull; int64_t k = h & (hcap - 1);
    if ((j > i && (k <= i || k > j)) || (j < i && (k <= i && k > j))) { htab[i] = htab[j]; hval[i] = hval[j]; htab[j] = -1; i = j; } } }
int64_t simulate(int64_t nrows, const int32_t *order, const int64_t *off, const int32_t *eid, int64_t W, int64_t cap_lines, int line_rows) {
  hcap = 1; while (hcap < cap_lines * 4) hcap <<= 1;
  htab = malloc(hcap * 8); hval = malloc(hcap * 4); memset(htab, 0xff, hcap * 8);
  Node *nd = malloc(sizeof(Node) * (cap_lines + 1)); int32_t head = -1, tail = -1, nfree = 0, used = 0;
  int64_t misses = 0;
  int64_t *cur = malloc(W * 8), *end = malloc(W * 8);
  for (int64_t r0 = 0; r0 < nrows; r0 += W) {
    int64_t n = nrows - r0 < W ? nrows - r0 : W, live = n;
    for (int64_t k = 0; k < n; k++) { int32_t r = order[r0 + k]; cur[k] = off[r]; end[k] = off[r + 1]; }
    while (live > 0) {
      live = 0;
      for (int64_t k = 0; k < n; k++) {
        if (cur[k] >= end[k]) continue; live++;
        int64_t line = eid[cur[k]++] / line_rows;
        int64_t hi = hfind(line);
        if (htab[hi] == line) { // hit: move to front
          int32_t x = hval[hi];
          if (x != head) { Node *q = &nd[x];
            if (q->prev >= 0) nd[q->prev].next = q->next; if (q->next >= 0) nd[q->next].prev = q->prev; else tail = q->prev;
            q->prev = -1; q->next = head; nd[head].prev = x; head = x; }
        } else {
          misses++;
          int32_t x;
          if (used < cap_lines) x = used++;
          else { x = tail; tail = nd[x].prev; nd[tail].next = -1; hdel(hfind(nd[x].key)); hi = hfind(line); }
          nd[x].key = line; nd[x].prev = -1; nd[x].next = head; if (head >= 0) nd[head].prev = x; head = x; if (tail < 0) tail = x;
          htab[hi] = line; hval[hi] = x;
        }
      }
    }
  }
  free(htab); free(hval); free(nd); free(cur); free(end);
  return misses;
}
// continuous: W slots; a slot that finishes its row pulls the next row of the schedule at once
int64_t simulate2(int64_t nrows, const int32_t *order, const int64_t *off, const int32_t *eid, int64_t W, int64_t cap_lines, int line_rows) {
  hcap = 1; while (hcap < cap_lines * 4) hcap <<= 1;
  htab = malloc(hcap * 8); hval = malloc(hcap * 4); memset(htab, 0xff, hcap * 8);
  Node *nd = malloc(sizeof(Node) * (cap_lines + 1)); int32_t head = -1, tail = -1, used = 0;
  int64_t misses = 0, next = 0, live = 0;
  int64_t *cur = malloc(W * 8), *end = malloc(W * 8);
  for (int64_t k = 0; k < W; k++) { cur[k] = end[k] = 0; }
  for (;;) {
    live = 0;
    for (int64_t k = 0; k < W; k++) {
      while (cur[k] >= end[k] && next < nrows) { int32_t r = order[next++]; cur[k] = off[r]; end[k] = off[r + 1]; }
      if (cur[k] >= end[k]) continue; live++;
      int64_t line = eid[cur[k]++] / line_rows;
      int64_t hi = hfind(line);
      if (htab[hi] == line) {
        int32_t x = hval[hi];
        if (x != head) { Node *q = &nd[x];
          if (q->prev >= 0) nd[q->prev].next = q->next; if (q->next >= 0) nd[q->next].prev = q->prev; else tail = q->prev;
          q->prev = -1; q->next = head; nd[head].prev = x; head = x; }
      } else {
        misses++;
        int32_t x;
        if (used < cap_lines) x = used++;
        else { x = tail; tail = nd[x].prev; nd[tail].next = -1; hdel(hfind(nd[x].key)); hi = hfind(line); }
        nd[x].key = line; nd[x].prev = -1; nd[x].next = head; if (head >= 0) nd[head].prev = x; head = x; if (tail < 0) tail = x;
        htab[hi] = line; hval[hi] = x;
      }
    }
    if (live == 0 && next >= nrows) break;
  }
  free(htab); free(hval); free(nd); free(cur); free(end);
  return misses;
}
