/*
 * hull_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker for the B200 kernels, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * it.  It restates, in plain C, the algorithm of the reference package
 * `hull3d` (arxiv/paper_1205_1171) for the path BASELINE.json names:
 *
 *   presort            pkg/src/hull3d/api.py:61-110   (_sort_and_perturb,
 *                                                      perturb_ties, _lex_order)
 *   event time          pkg/src/hull3d/_ckernels.pyx:34-46   (_evtime)
 *   toggle              pkg/src/hull3d/_ckernels.pyx:49-60   (_act)
 *   bridge at -inf      pkg/src/hull3d/_ckernels.pyx:63-83   (_find_bridge)
 *   pairwise merge      pkg/src/hull3d/_ckernels.pyx:86-208  (_merge_one)
 *   level plan / loop   pkg/src/hull3d/parallel.py:27-112    (plan_level, build_movie)
 *   carry copy          pkg/src/hull3d/_ckernels.pyx:363-375 (copy_log)
 *   facet extraction    pkg/src/hull3d/_ckernels.pyx:324-349 (extract_faces)
 *
 * Arithmetic contract: fp64, no FMA contraction (the reference builds with
 * -ffp-contract=off, pkg/setup.py:51-54); the Makefile passes the same flag.
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref, built by oracle/build_ref.sh) through tests/golden/ fixtures
 * and tests/test_oracle_*.py.
 *
 * Data model (pkg/src/hull3d/store.py:46-118): P = n rows of (x,y,z) f64,
 * K = n rows of (prev,next) i32, logs = flat i32 buffers of 2n slots with
 * the log of group [L,R) at slot 2L, NIL-terminated.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_NIL (-1)
#define ORC_E_OVERFLOW (-1)
#define ORC_E_BRIDGE (-2)
#define ORC_E_CHAIN (-3)
#define ORC_E_COUNT (-4)
#define ORC_E_UNTERMINATED (-5)

typedef int64_t i64;
typedef int32_t i32;

#define PX(i) P[3 * (i)]
#define PY(i) P[3 * (i) + 1]
#define PZ(i) P[3 * (i) + 2]
#define PREV(i) K[2 * (i)]
#define NEXT(i) K[2 * (i) + 1]

/* Time at which the kinetic projections (x, z - t*y) of a, b, c are
 * collinear; +inf if any index is NIL or the xy-determinant is exactly 0.
 * Operand order follows _ckernels.pyx:34-46 (base point a, den tested first). */
double orc_evtime(const double *P, i64 a, i64 b, i64 c) {
    if (a == ORC_NIL || b == ORC_NIL || c == ORC_NIL) return INFINITY;
    const double ax = PX(a), ay = PY(a);
    const double dbx = PX(b) - ax;
    const double dcx = PX(c) - ax;
    const double det_xy = dbx * (PY(c) - ay) - dcx * (PY(b) - ay);
    if (det_xy == 0.0) return INFINITY;
    const double az = PZ(a);
    const double det_xz = dbx * (PZ(c) - az) - dcx * (PZ(b) - az);
    return det_xz / det_xy;
}

/* Toggle point i in the chain: splice it between its recorded neighbours
 * unless they already link through it, in which case unlink it.  i's own
 * links are never written.  -1 on a NIL neighbour (_ckernels.pyx:49-60). */
int orc_act(i32 *K, i64 i) {
    const i64 lft = PREV(i), rgt = NEXT(i);
    if (lft == ORC_NIL || rgt == ORC_NIL) return -1;
    if (NEXT(lft) == i) {          /* currently linked: delete */
        NEXT(lft) = (i32)rgt;
        PREV(rgt) = (i32)lft;
    } else {                       /* parked: insert */
        NEXT(lft) = (i32)i;
        PREV(rgt) = (i32)i;
    }
    return 0;
}

/* Lower common tangent of two adjacent chains at t = -inf: advance the right
 * foot while the xy-turn (u, v, next v) is clockwise, otherwise retreat the
 * left foot while (prev u, u, v) is clockwise (_ckernels.pyx:63-83). */
i64 orc_find_bridge(const double *P, const i32 *K, i64 *pu, i64 *pv, i64 limit) {
    i64 u = *pu, v = *pv, moves = 0;
    for (;;) {
        const i64 vn = NEXT(v);
        int moved = 0;
        if (vn != ORC_NIL &&
            (PX(v) - PX(u)) * (PY(vn) - PY(u)) - (PX(vn) - PX(u)) * (PY(v) - PY(u)) < 0.0) {
            v = vn;
            moved = 1;
        } else {
            const i64 up = PREV(u);
            if (up != ORC_NIL &&
                (PX(u) - PX(up)) * (PY(v) - PY(up)) - (PX(v) - PX(up)) * (PY(u) - PY(up)) < 0.0) {
                u = up;
                moved = 1;
            }
        }
        if (!moved) {
            *pu = u;
            *pv = v;
            return 0;
        }
        if (++moves > limit) return ORC_E_BRIDGE;
    }
}

/* Emit one event into the output slice, with the overflow guard that
 * precedes every write in _merge_one (k >= cap-1, _ckernels.pyx:143). */
#define EMIT(e)                                   \
    do {                                          \
        if (k >= cap - 1) return ORC_E_OVERFLOW;  \
        out[base + k] = (i32)(e);                 \
        ++k;                                      \
    } while (0)

/* Merge the movies of [L,M) and [M,R): the kinetic sweep over six candidate
 * events (two child events, four bridge-foot moves), then stitch, then the
 * backward rewind that leaves the chain at the merged start-of-time state.
 * Returns the merged event count or a negative code (_ckernels.pyx:86-208). */
i64 orc_merge(const double *P, i32 *K, const i32 *in, i32 *out, i64 L, i64 M, i64 R) {
    const i64 cap = 2 * (R - L);
    const i64 base = 2 * L;
    i64 u = M - 1, v = M;
    i64 li = 2 * L, ri = 2 * M;
    const i64 lend = 2 * M, rend = 2 * R;
    i64 k = 0;
    double tcur = -INFINITY;

    if (orc_find_bridge(P, K, &u, &v, R - L) < 0) return ORC_E_BRIDGE;

    for (;;) {
        if (li >= lend || ri >= rend) return ORC_E_UNTERMINATED;
        const i64 el = in[li], er = in[ri];
        double cand[6];
        cand[0] = (el != ORC_NIL) ? orc_evtime(P, PREV(el), el, NEXT(el)) : INFINITY;
        cand[1] = (er != ORC_NIL) ? orc_evtime(P, PREV(er), er, NEXT(er)) : INFINITY;
        cand[2] = orc_evtime(P, u, NEXT(u), v);
        cand[3] = orc_evtime(P, PREV(u), u, v);
        cand[4] = orc_evtime(P, u, v, NEXT(v));
        cand[5] = orc_evtime(P, u, PREV(v), v);
        /* earliest candidate strictly after tcur; ties go to the lowest case */
        double best = INFINITY;
        int which = -1;
        for (int c = 0; c < 6; ++c) {
            if (cand[c] > tcur && cand[c] < best) {
                best = cand[c];
                which = c;
            }
        }
        if (which < 0) break;
        switch (which) {
        case 0:
            if (PX(el) < PX(u)) EMIT(el);
            if (orc_act(K, el) < 0) return ORC_E_CHAIN;
            ++li;
            break;
        case 1:
            if (PX(er) > PX(v)) EMIT(er);
            if (orc_act(K, er) < 0) return ORC_E_CHAIN;
            ++ri;
            break;
        case 2:
            u = NEXT(u);
            EMIT(u);
            break;
        case 3:
            EMIT(u);
            u = PREV(u);
            break;
        case 4:
            EMIT(v);
            v = NEXT(v);
            break;
        default:
            v = PREV(v);
            EMIT(v);
            break;
        }
        tcur = best;
    }

    out[base + k] = ORC_NIL;
    NEXT(u) = (i32)v;          /* final bridge at t = +inf */
    PREV(v) = (i32)u;

    for (i64 idx = k - 1; idx >= 0; --idx) {
        const i64 e = out[base + idx];
        if (PX(e) <= PX(u) || PX(e) >= PX(v)) {
            if (orc_act(K, e) < 0) return ORC_E_CHAIN;
            if (e == u)
                u = PREV(u);
            else if (e == v)
                v = NEXT(v);
        } else {               /* e was a bridge foot: splice it back */
            NEXT(u) = (i32)e;
            PREV(e) = (i32)u;
            PREV(v) = (i32)e;
            NEXT(e) = (i32)v;
            if (e < M)
                u = e;
            else
                v = e;
        }
    }
    return k;
}

/* Every point is a one-point hull with an empty log at slot 2i
 * (_ckernels.pyx:237-245). */
void orc_init_base(i32 *K, i32 *slots, i64 n) {
    for (i64 i = 0; i < n; ++i) {
        PREV(i) = ORC_NIL;
        NEXT(i) = ORC_NIL;
        slots[2 * i] = ORC_NIL;
    }
}

/* Copy a NIL-terminated log slice (_ckernels.pyx:363-375). */
i64 orc_copy_log(const i32 *src, i32 *dst, i64 off, i64 cap) {
    for (i64 idx = 0; idx < cap; ++idx) {
        dst[off + idx] = src[off + idx];
        if (src[off + idx] == ORC_NIL) return idx;
    }
    return ORC_E_UNTERMINATED;
}

i64 orc_level_count(i64 n) {
    i64 lv = 0;
    while ((((i64)1) << lv) < n) ++lv;
    return lv;
}

/* One level of plan_level + build_movie (parallel.py:49-65, :96-111): groups
 * of 2^level points; a group with more than half a group of points is a
 * merge job, the trailing short group is carried.  Optionally records the
 * merged length of every job into kout[group]. */
i64 orc_run_level(const double *P, i64 n, i32 *K, const i32 *in, i32 *out, i64 level, i64 *kout) {
    const i64 size = ((i64)1) << level, half = size >> 1;
    for (i64 L = 0, g = 0; L < n; L += size, ++g) {
        const i64 R = (L + size < n) ? L + size : n;
        i64 r;
        if (R - L > half) {
            r = orc_merge(P, K, in, out, L, L + half, R);
        } else {
            r = orc_copy_log(in, out, 2 * L, 2 * n - 2 * L);
        }
        if (r < 0) return r;
        if (kout) kout[g] = r;
    }
    return 0;
}

/* Full bottom-up build; returns 0 if the final log is in bufA, 1 if in bufB,
 * or a negative code. */
i64 orc_build_movie(const double *P, i64 n, i32 *K, i32 *bufA, i32 *bufB) {
    orc_init_base(K, bufA, n);
    i32 *src = bufA, *dst = bufB;
    int in_b = 0;
    const i64 levels = orc_level_count(n);
    for (i64 lv = 1; lv <= levels; ++lv) {
        const i64 r = orc_run_level(P, n, K, src, dst, lv, NULL);
        if (r < 0) return r;
        i32 *t = src;
        src = dst;
        dst = t;
        in_b ^= 1;
    }
    return in_b;
}

/* Replay the log from its start-of-time chain, recording (prev, e, next)
 * before each toggle (_ckernels.pyx:324-349).  Returns the facet count. */
i64 orc_extract_faces(i32 *K, const i32 *slots, i64 off, i32 *faces, i64 limit) {
    i64 m = 0;
    for (i64 idx = off;; ++idx) {
        const i64 e = slots[idx];
        if (e == ORC_NIL) return m;
        if (m >= limit) return ORC_E_OVERFLOW;
        faces[3 * m] = PREV(e);
        faces[3 * m + 1] = (i32)e;
        faces[3 * m + 2] = NEXT(e);
        if (orc_act(K, e) < 0) return ORC_E_CHAIN;
        ++m;
    }
}

/* Replay forward / backward (_ckernels.pyx:292-321). */
i64 orc_replay(i32 *K, const i32 *slots, i64 off, i64 count, int backward) {
    for (i64 s = 0; s < count; ++s) {
        const i64 e = slots[off + (backward ? count - 1 - s : s)];
        if (e == ORC_NIL) return ORC_E_COUNT;
        if (orc_act(K, e) < 0) return ORC_E_CHAIN;
    }
    return 0;
}

/* One whole pass: build + extract.  Returns the facet count (faces must hold
 * 2n triples) or a negative code.  The caller passes z already negated for
 * the upper pass (api.py:215-216). */
i64 orc_hull_pass(const double *P, i64 n, i32 *faces, i64 limit) {
    i32 *K = (i32 *)malloc(sizeof(i32) * 2 * (size_t)n);
    i32 *A = (i32 *)malloc(sizeof(i32) * 2 * (size_t)n);
    i32 *B = (i32 *)malloc(sizeof(i32) * 2 * (size_t)n);
    i64 r = -100;
    if (K && A && B) {
        for (i64 s = 0; s < 2 * n; ++s) A[s] = B[s] = ORC_NIL;
        r = orc_build_movie(P, n, K, A, B);
        if (r >= 0) r = orc_extract_faces(K, r ? B : A, 0, faces, limit);
    }
    free(K);
    free(A);
    free(B);
    return r;
}

/* ---------------------------------------------------------------- presort */

typedef struct {
    const double *P;
    int lex; /* 0: key x only; 1: (x, y, z) */
} orc_cmp_ctx;

/* three-way compare of rows a, b; equal keys fall back to the index so the
 * sort is stable (numpy argsort kind="stable", lexsort are both stable).
 * -0.0 == +0.0 under C comparison, as under numpy's. */
static int orc_row_cmp(const orc_cmp_ctx *c, i64 a, i64 b) {
    const double *P = c->P;
    const int ncols = c->lex ? 3 : 1;
    for (int col = 0; col < ncols; ++col) {
        const double da = P[3 * a + col], db = P[3 * b + col];
        if (da < db) return -1;
        if (db < da) return 1;
    }
    return (a < b) ? -1 : (a > b);
}

static void orc_msort(const orc_cmp_ctx *c, i64 *idx, i64 *tmp, i64 n) {
    if (n < 2) return;
    const i64 h = n / 2;
    orc_msort(c, idx, tmp, h);
    orc_msort(c, idx + h, tmp, n - h);
    i64 a = 0, b = h, o = 0;
    while (a < h && b < n) tmp[o++] = (orc_row_cmp(c, idx[b], idx[a]) < 0) ? idx[b++] : idx[a++];
    while (a < h) tmp[o++] = idx[a++];
    while (b < n) tmp[o++] = idx[b++];
    memcpy(idx, tmp, sizeof(i64) * (size_t)n);
}

/* Restates _sort_and_perturb (api.py:90-110) with perturb_ties (api.py:61-83):
 * stable argsort of x; if x has any adjacent tie, lexsort (x,y,z), nudge each
 * tie run by rank*16eps*max(1,|base|), stable re-sort and re-check.
 * Writes sorted rows and the permutation; returns 0 (no ties), 1 (perturbed),
 * or -6 if duplicate x survive perturbation (DegenerateInputError). */
int orc_sort_and_perturb(const double *pts, i64 n, double *sorted, i64 *order) {
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *tmp = (i64 *)malloc(sizeof(i64) * (size_t)n);
    double *work = (double *)malloc(sizeof(double) * 3 * (size_t)n);
    int ret = 0;
    orc_cmp_ctx c = {pts, 0};
    for (i64 i = 0; i < n; ++i) idx[i] = i;
    orc_msort(&c, idx, tmp, n);
    int tie = 0;
    for (i64 i = 1; i < n && !tie; ++i) tie = !(pts[3 * idx[i]] > pts[3 * idx[i - 1]]);
    if (!tie) {
        for (i64 i = 0; i < n; ++i) {
            order[i] = idx[i];
            memcpy(sorted + 3 * i, pts + 3 * idx[i], 3 * sizeof(double));
        }
        goto done;
    }
    c.lex = 1;
    for (i64 i = 0; i < n; ++i) idx[i] = i;
    orc_msort(&c, idx, tmp, n);
    for (i64 i = 0; i < n; ++i) memcpy(work + 3 * i, pts + 3 * idx[i], 3 * sizeof(double));
    {
        const double tie_eps = 16.0 * 2.220446049250313080847263336181640625e-16;
        i64 i = 0;
        while (i < n) {
            i64 j = i + 1;
            while (j < n && work[3 * j] == work[3 * i]) ++j;
            if (j - i > 1) {
                const double x0 = work[3 * i];
                const double ax = fabs(x0);
                const double step = tie_eps * (ax > 1.0 ? ax : 1.0);
                for (i64 r = 1; r < j - i; ++r) work[3 * (i + r)] = x0 + (double)r * step;
            }
            i = j;
        }
    }
    /* stable re-sort of the perturbed x; suborder composes with the lexsort */
    {
        orc_cmp_ctx c2 = {work, 0};
        i64 *sub = (i64 *)malloc(sizeof(i64) * (size_t)n);
        for (i64 i = 0; i < n; ++i) sub[i] = i;
        orc_msort(&c2, sub, tmp, n);
        for (i64 i = 0; i < n; ++i) {
            order[i] = idx[sub[i]];
            memcpy(sorted + 3 * i, work + 3 * sub[i], 3 * sizeof(double));
        }
        free(sub);
    }
    ret = 1;
    for (i64 i = 1; i < n; ++i)
        if (!(sorted[3 * i] > sorted[3 * (i - 1)])) {
            ret = -6;
            break;
        }
done:
    free(idx);
    free(tmp);
    free(work);
    return ret;
}
