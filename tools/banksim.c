// banksim.c -- shared-memory bank-conflict simulator for the quad-layout
// chunk stream (lane runs), used to design the column-order optimizer of
// stream_build (csrc/rsr_preprocess.cu).  One random ternary cell (k rows,
// tn columns, P(0) = 1/2) is laid out exactly like the device builder; the
// cost of one gather instruction (round r, slot s) is the max over the 32
// banks of the number of distinct addresses the active lanes read.
//
//   gcc -O2 -o /tmp/banksim tools/banksim.c -lm && /tmp/banksim [tn] [k] [cells] [passes]
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t rs = 88172645463325252ull;
static uint64_t xr(void) { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return rs; }

typedef struct { int key, n, *cols; int *pos; } Group;

static int tn = 16384, K = 6, NB = 32;
static int BMODE = 0;   // 0: 4-byte v (bank c%32), 1: 2-byte v (bank (c/2)%32)
static int PADFREE = 0; // 1: pads read a zero word in any bank (chosen least loaded)
static inline int bank_of(int c) { return BMODE ? (c >> 1) & 31 : c & 31; }
static int *ent;        // logical slot -> column (>=0), or -1 key, -2 pad (column 0)
static int nslots, npairs, P, Lf, rem_;
static int *load;       // [round][slot][bank] distinct-address counts (pads: flag)
static int *padc;       // [round][slot] pads (address 0) present

static inline void slot_rs(int p, int *r, int *s, int *lane) {
    int j = p >> 5;
    *lane = j / P;
    *r = j - *lane * P;
    *s = p & 31;
}

static int inst_cost(int r, int s) {
    int *l = load + ((size_t)r * 32 + s) * NB;
    int m = 0;
    for (int b = 0; b < NB; ++b) {
        int x = l[b] + (b == 0 && padc[r * 32 + s] ? 1 : 0);
        if (x > m) m = x;
    }
    return m ? m : 1;
}

static double total_cost(double *lb) {
    long tot = 0, ninst = 0, lbt = 0;
    for (int r = 0; r < P; ++r) {
        int tb[64] = {0};
        for (int s = 1; s < 32; ++s) {
            tot += inst_cost(r, s);
            ++ninst;
            for (int b = 0; b < NB; ++b) tb[b] += load[((size_t)r * 32 + s) * NB + b];
            if (padc[r * 32 + s]) tb[0] += 1;
        }
        int mb = 31;
        for (int b = 0; b < NB; ++b) if (tb[b] > mb) mb = tb[b];
        lbt += mb;
    }
    *lb = (double)lbt / ninst;
    return (double)tot / ninst;
}

// ---- Hungarian algorithm (min cost, n x n), classic O(n^3)
static double hung(int n, const double *a, int *assign) {
    static double u[512], v[512], minv[512];
    static int p[512], way[512], used[512];
    for (int i = 0; i <= n; ++i) { u[i] = v[i] = 0; p[i] = way[i] = 0; }
    for (int i = 1; i <= n; ++i) {
        p[0] = i;
        int j0 = 0;
        for (int j = 0; j <= n; ++j) { minv[j] = 1e18; used[j] = 0; }
        do {
            used[j0] = 1;
            int i0 = p[j0], j1 = 0;
            double delta = 1e18;
            for (int j = 1; j <= n; ++j)
                if (!used[j]) {
                    double cur = a[(i0 - 1) * n + (j - 1)] - u[i0] - v[j];
                    if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
                    if (minv[j] < delta) { delta = minv[j]; j1 = j; }
                }
            for (int j = 0; j <= n; ++j)
                if (used[j]) { u[p[j]] += delta; v[j] -= delta; }
                else minv[j] -= delta;
            j0 = j1;
        } while (p[j0] != 0);
        do { int j1 = way[j0]; p[j0] = p[j1]; j0 = j1; } while (j0);
    }
    for (int j = 1; j <= n; ++j) assign[p[j] - 1] = j - 1;  // row -> col
    return -v[0];
}

static double W_MAX = 64.0;  // weight of raising an instruction's max load
static int ALG = 0;
static int PREFER = 0;
static int NOBFS = 0;
static int NOORDER = 0;           // 0: Hungarian coordinate descent, 1: pairwise swaps

static double inst_obj(int r, int s) {
    int *l = load + ((size_t)r * 32 + s) * NB;
    int m = 0;
    double sq = 0;
    for (int b = 0; b < NB; ++b) {
        int x = l[b] + (b == 0 && padc[r * 32 + s] ? 1 : 0);
        if (x > m) m = x;
        sq += (double)x * x;
    }
    return W_MAX * m + sq;
}

// marginal cost of adding one address of bank b at (r, s)
static double marg(int r, int s, int b) {
    int *l = load + ((size_t)r * 32 + s) * NB;
    int m = 0;
    for (int bb = 0; bb < NB; ++bb) {
        int x = l[bb] + (bb == 0 && padc[r * 32 + s] ? 1 : 0);
        if (x > m) m = x;
    }
    int x = l[b] + (b == 0 && padc[r * 32 + s] ? 1 : 0);
    double d = (x + 1 > m ? W_MAX : 0.0) + (double)(2 * x + 1);
    return d;
}

int main(int argc, char **argv) {
    if (argc > 1) tn = atoi(argv[1]);
    if (argc > 2) K = atoi(argv[2]);
    int cells = argc > 3 ? atoi(argv[3]) : 3;
    int passes = argc > 4 ? atoi(argv[4]) : 4;
    if (argc > 5) W_MAX = atof(argv[5]);
    if (argc > 6) BMODE = atoi(argv[6]);
    if (argc > 7) PADFREE = atoi(argv[7]);
    if (argc > 8) ALG = atoi(argv[8]);
    if (argc > 9) PREFER = atoi(argv[9]);
    if (argc > 10) NOBFS = atoi(argv[10]);
    if (argc > 11) NOORDER = atoi(argv[11]);
    int nk = 1;
    for (int i = 0; i < K; ++i) nk *= 3;
    for (int cell = 0; cell < cells; ++cell) {
        // keys
        int *key = malloc(sizeof(int) * tn);
        for (int c = 0; c < tn; ++c) {
            int kk = 0, p3 = 1;
            for (int i = 0; i < K; ++i) {
                uint64_t u = xr() & 3;  // 0,1 -> 0; 2 -> +1; 3 -> -1
                int d = u < 2 ? 0 : (u == 2 ? 1 : 2);
                kk += d * p3;
                p3 *= 3;
            }
            key[c] = kk;
        }
        int *cnt = calloc(nk, sizeof(int));
        for (int c = 1; c < tn; ++c) cnt[key[c]]++;  // column 0 travels as col0_key
        int G = 0;
        for (int kk = 1; kk < nk; ++kk) G += cnt[kk] > 0;
        Group *g = calloc(G, sizeof(Group));
        int *gi = malloc(sizeof(int) * nk);
        for (int kk = 1, x = 0; kk < nk; ++kk) {
            gi[kk] = -1;
            if (cnt[kk]) { g[x].key = kk; g[x].cols = malloc(sizeof(int) * cnt[kk]);
                           g[x].pos = malloc(sizeof(int) * cnt[kk]); gi[kk] = x++; }
        }
        for (int c = 1; c < tn; ++c) if (key[c]) { Group *q = &g[gi[key[c]]]; q->cols[q->n++] = c; }
        // quad layout
        int cap = tn * 2 + 64 * G;
        ent = malloc(sizeof(int) * cap);
        int p = 0;
        for (int x = 0; x < G; ++x) {
            ent[p++] = -1;
            for (int j = 0; j < g[x].n; ++j) {
                if ((p & 31) == 0) ent[p++] = -1;
                g[x].pos[j] = p;
                ent[p++] = g[x].cols[j];
            }
            while (p & 3) ent[p++] = -2;
        }
        while (p & 31) ent[p++] = (p & 3) ? -2 : -1;
        nslots = p;
        npairs = p / 32;
        P = (npairs + 31) / 32;
        Lf = npairs / P;
        rem_ = npairs - Lf * P;
        load = calloc((size_t)P * 32 * NB, sizeof(int));
        padc = calloc((size_t)P * 32, sizeof(int));
#define REBUILD()                                                                 \
        do {                                                                      \
            memset(load, 0, sizeof(int) * (size_t)P * 32 * NB);                   \
            memset(padc, 0, sizeof(int) * (size_t)P * 32);                        \
            for (int q = 0; q < nslots; ++q) {                                    \
                int r, s, ln;                                                     \
                slot_rs(q, &r, &s, &ln);                                          \
                if (ent[q] >= 0) load[((size_t)r * 32 + s) * NB + bank_of(ent[q])]++; \
                else if (!PADFREE && (ent[q] == -2 || ((q & 3) && ent[q] == -1))) padc[r * 32 + s] = 1; \
            }                                                                     \
            for (int r = 0; r < P; ++r) {                                         \
                int np = Lf + (r < rem_);                                         \
                if (np < 32 && !PADFREE) for (int s = 1; s < 32; ++s) padc[r * 32 + s] = 1;   \
            }                                                                     \
        } while (0)
        REBUILD();
        double lb, c0 = total_cost(&lb);
        // greedy: per group in order, each position takes the least-loaded bank column
        for (int x = 0; x < G; ++x) {
            int n = g[x].n;
            int *rest = malloc(sizeof(int) * n);
            memcpy(rest, g[x].cols, sizeof(int) * n);
            for (int j = 0; j < n; ++j) {
                int q = g[x].pos[j], r, s, ln;
                slot_rs(q, &r, &s, &ln);
                int old = ent[q];
                load[((size_t)r * 32 + s) * NB + bank_of(old)]--;
                int best = -1, bl = 1 << 30;
                for (int t = j; t < n; ++t) {
                    int l = load[((size_t)r * 32 + s) * NB + bank_of(rest[t])];
                    if (l < bl) { bl = l; best = t; }
                }
                int c = rest[best]; rest[best] = rest[j]; rest[j] = c;
                ent[q] = c;
                load[((size_t)r * 32 + s) * NB + bank_of(c)]++;
            }
            free(rest);
        }
        if (ALG >= 3) {
            // instruction-wise maximum matching: slots (r, s) in order; each lane
            // whose slot is a column takes one unplaced column of its group, banks
            // distinct across lanes where a matching allows (Kuhn's algorithm)
            int *grp_of = malloc(sizeof(int) * nslots);
            for (int q = 0; q < nslots; ++q) grp_of[q] = -1;
            for (int x = 0; x < G; ++x) for (int j = 0; j < g[x].n; ++j) grp_of[g[x].pos[j]] = x;
            int **pool = malloc(sizeof(int *) * G);
            int *pn = malloc(sizeof(int) * G);
            for (int x = 0; x < G; ++x) { pool[x] = malloc(sizeof(int) * g[x].n); memcpy(pool[x], g[x].cols, sizeof(int) * g[x].n); pn[x] = g[x].n; }
            memset(load, 0, sizeof(int) * (size_t)P * 32 * NB);
            for (int r = 0; r < P; ++r) {
                int np = Lf + (r < rem_);
                for (int s = 1; s < 32; ++s) {
                    int lanes[32], nl = 0;
                    for (int L = 0; L < np; ++L) {
                        int q = (L * P + r) * 32 + s;
                        if (q < nslots && grp_of[q] >= 0) lanes[nl++] = L;
                    }
                    // candidate banks per lane, by multiplicity in the pool
                    int cntb[32][32];
                    for (int i = 0; i < nl; ++i) {
                        int x = grp_of[(lanes[i] * P + r) * 32 + s];
                        memset(cntb[i], 0, sizeof(cntb[i]));
                        for (int t = 0; t < pn[x]; ++t) cntb[i][bank_of(pool[x][t])]++;
                    }
                    int bank_lane[32], lane_bank[32];
                    for (int b = 0; b < 32; ++b) bank_lane[b] = -1;
                    for (int i = 0; i < nl; ++i) lane_bank[i] = -1;
                    // Kuhn: try augmenting from each lane (fewest options first)
                    int order[32];
                    for (int i = 0; i < nl; ++i) order[i] = i;
                    for (int a = 0; a < (NOORDER ? 0 : nl); ++a) for (int b2 = a + 1; b2 < nl; ++b2) {
                        int da = 0, db = 0;
                        for (int b = 0; b < 32; ++b) { da += cntb[order[a]][b] > 0; db += cntb[order[b2]][b] > 0; }
                        if (db < da) { int t = order[a]; order[a] = order[b2]; order[b2] = t; }
                    }
                    for (int oi = 0; oi < nl; ++oi) {
                        int i0 = order[oi];
                        int vis[32] = {0};
                        // DFS with explicit recursion via lambda-like helper
                        int stack_i[64], stack_b[64], sp = 0;
                        int found = 0;
                        // iterative DFS: try banks of lane i in descending multiplicity
                        int prevb[32]; for (int b = 0; b < 32; ++b) prevb[b] = -2;
                        int qi[64], qh = 0, qt = 0; qi[qt++] = i0;
                        int parent_lane[32]; for (int b = 0; b < 32; ++b) parent_lane[b] = -1;
                        int endb = -1;
                        if (PREFER == 1) {  // a free bank first, the pool's most abundant one
                            int bb = -1, bc = 0;
                            for (int b = 0; b < 32; ++b)
                                if (cntb[i0][b] > bc && bank_lane[b] < 0) { bc = cntb[i0][b]; bb = b; }
                            if (bb >= 0) { vis[bb] = 1; parent_lane[bb] = i0; endb = bb; found = 1; }
                        } else if (PREFER >= 2) {  // O(1): a free bank holding >= 2 columns, else any free
                            int bb = -1;
                            for (int pass = 0; pass < 2 && bb < 0; ++pass)
                                for (int t = 0; t < 32; ++t) {
                                    int b = (t + (PREFER == 3 ? 7 * i0 : 0)) & 31;
                                    if (bank_lane[b] < 0 && cntb[i0][b] >= (pass == 0 ? 2 : 1)) { bb = b; break; }
                                }
                            if (bb >= 0) { vis[bb] = 1; parent_lane[bb] = i0; endb = bb; found = 1; }
                        }
                        while (!NOBFS && qh < qt && !found) {
                            int i = qi[qh++];
                            for (int pass = 0; pass < 2 && !found; ++pass)
                            for (int b = 0; b < 32; ++b) {
                                if (!cntb[i][b] || vis[b]) continue;
                                vis[b] = 1; parent_lane[b] = i;
                                if (bank_lane[b] < 0) { endb = b; found = 1; break; }
                                qi[qt++] = bank_lane[b];
                            }
                        }
                        (void)stack_i; (void)stack_b; (void)sp; (void)prevb;
                        if (found) {
                            int b = endb;
                            while (b >= 0) {
                                int i = parent_lane[b];
                                int ob = lane_bank[i];
                                lane_bank[i] = b; bank_lane[b] = i;
                                b = ob;
                                if (i == i0) break;
                            }
                        }
                    }
                    int f32l[32] = {0};
                    for (int i = 0; i < nl; ++i) {
                        int q = (lanes[i] * P + r) * 32 + s;
                        int x = grp_of[q];
                        int b = lane_bank[i];
                        int t = 0;
                        if (b >= 0) {  // among the bank's columns: the least-used f32 bank
                            int bl = 1 << 30;
                            for (int u = 0; u < pn[x]; ++u)
                                if (bank_of(pool[x][u]) == b) {
                                    int l = f32l[(BMODE ? pool[x][u] : pool[x][u] >> 1) & 31];
                                    if (l < bl) { bl = l; t = u; }
                                }
                            f32l[(BMODE ? pool[x][t] : pool[x][t] >> 1) & 31]++;
                        }
                        else {  // unmatched: the column whose bank is least loaded here
                            int bl = 1 << 30;
                            for (int u = 0; u < pn[x]; ++u) { int l = load[((size_t)r * 32 + s) * NB + bank_of(pool[x][u])]; if (l < bl) { bl = l; t = u; } }
                        }
                        int c = pool[x][t]; pool[x][t] = pool[x][--pn[x]];
                        ent[q] = c;
                        load[((size_t)r * 32 + s) * NB + bank_of(c)]++;
                    }
                }
            }
            for (int x = 0; x < G; ++x) free(pool[x]);
            free(pool); free(pn); free(grp_of);
            if (ALG == 4) ALG = 1; else if (ALG == 5) ALG = 0; else passes = 0;
        }
        // positions keep the greedy layout's column slots; loads now reflect greedy
        double c1 = total_cost(&lb);
        // coordinate descent: optimal reassignment of each group's columns
        double *A = malloc(sizeof(double) * 512 * 512);
        int *asg = malloc(sizeof(int) * 512);
        double cp[16];
        for (int pass = 0; pass < passes; ++pass) {
            for (int x = 0; x < G; ++x) {
                int n = g[x].n;
                if (n < 2 || n > 512) continue;
                if (ALG == 1) {
                    for (int i = 0; i < n; ++i)
                        for (int j = i + 1; j < n; ++j) {
                            int q1 = g[x].pos[i], q2 = g[x].pos[j], r1, s1, r2, s2, ln;
                            slot_rs(q1, &r1, &s1, &ln);
                            slot_rs(q2, &r2, &s2, &ln);
                            if (r1 == r2 && s1 == s2) continue;
                            int b1 = bank_of(ent[q1]), b2 = bank_of(ent[q2]);
                            if (b1 == b2) continue;
                            int *l1 = load + ((size_t)r1 * 32 + s1) * NB, *l2 = load + ((size_t)r2 * 32 + s2) * NB;
                            double o = inst_obj(r1, s1) + inst_obj(r2, s2);
                            l1[b1]--; l1[b2]++; l2[b2]--; l2[b1]++;
                            double nw = inst_obj(r1, s1) + inst_obj(r2, s2);
                            if (nw < o) { int t = ent[q1]; ent[q1] = ent[q2]; ent[q2] = t; }
                            else { l1[b1]++; l1[b2]--; l2[b2]++; l2[b1]--; }
                        }
                    continue;
                }
                int cols[512];
                for (int j = 0; j < n; ++j) {
                    int q = g[x].pos[j], r, s, ln;
                    slot_rs(q, &r, &s, &ln);
                    cols[j] = ent[q];
                    load[((size_t)r * 32 + s) * NB + bank_of(ent[q])]--;
                }
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < n; ++j) {
                        int q = g[x].pos[j], r, s, ln;
                        slot_rs(q, &r, &s, &ln);
                        A[i * n + j] = marg(r, s, bank_of(cols[i]));
                    }
                if (ALG == 2) {  // greedy assignment: cheapest (column, slot) pair first
                    static int ur[512], uc[512];
                    for (int i = 0; i < n; ++i) ur[i] = uc[i] = 0;
                    for (int t = 0; t < n; ++t) {
                        double best = 1e18; int bi = -1, bj = -1;
                        for (int i = 0; i < n; ++i) if (!ur[i])
                            for (int j = 0; j < n; ++j) if (!uc[j] && A[i * n + j] < best) { best = A[i * n + j]; bi = i; bj = j; }
                        ur[bi] = uc[bj] = 1; asg[bi] = bj;
                        // recompute the marginal costs of the chosen slot's instruction for the remaining columns
                        int q = g[x].pos[bj], r, s, ln;
                        slot_rs(q, &r, &s, &ln);
                        load[((size_t)r * 32 + s) * NB + bank_of(cols[bi])]++;
                        for (int i = 0; i < n; ++i) if (!ur[i]) A[i * n + bj] = marg(r, s, bank_of(cols[i]));
                        load[((size_t)r * 32 + s) * NB + bank_of(cols[bi])]--;
                    }
                } else hung(n, A, asg);
                for (int i = 0; i < n; ++i) {
                    int q = g[x].pos[asg[i]], r, s, ln;
                    slot_rs(q, &r, &s, &ln);
                    ent[q] = cols[i];
                    load[((size_t)r * 32 + s) * NB + bank_of(cols[i])]++;
                }
            }
            cp[pass] = total_cost(&lb);
        }
        printf("cell %d: groups %d pairs %d rounds %d | sorted %.3f greedy %.3f |", cell, G, npairs,
               P, c0, c1);
        for (int pass = 0; pass < passes; ++pass) printf(" cd%d %.3f", pass + 1, cp[pass]);
        printf(" | per-round lower bound %.3f", lb);
        {   int bm = BMODE; BMODE = !BMODE; REBUILD(); double lb2; double cx = total_cost(&lb2);
            printf(" | other bank map %.3f\n", cx); BMODE = bm; }
        free(A); free(asg);
        for (int x = 0; x < G; ++x) { free(g[x].cols); free(g[x].pos); }
        free(g); free(gi); free(cnt); free(key); free(ent); free(load); free(padc);
    }
    return 0;
}
