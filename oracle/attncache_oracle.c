/*
 * attncache_oracle.c — plain, slow, obviously-correct CPU oracle for the
 * AttnCache hot path (arXiv 2510.25979).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no source, header, table or helper with the CUDA library under
 * paper_2510_25979_b200/ and never includes or links it.
 *
 * Everything is accumulated in fp64 from the exact stored bytes (fp32, fp16
 * or bf16, decoded exactly).  No blocking, fusion or reordering beyond the
 * definitions below.  Paper line numbers refer to PAPER.md (the paper's
 * LaTeX source):
 *
 *   search  — Alg. 1 l.255-257 and PAPER.md:341:
 *             "(idx, sims) <- VecDB.search(f)"; "IF sims >= theta".
 *             sims is the inner product of L2-normalised feature vectors
 *             (BASELINE.json north_star; reading R1); top-1 with the
 *             lowest index among equal scores (north_star; reading R3); the
 *             gate is inclusive (">=", "not less than").
 *   apply   — Alg. 2 l.373-375: "h <- mat_mul(attn_map, v)"
 *             i.e. O = A . V, written as the plain matrix product over every
 *             column of A (the stored upper triangle is exact zeros).
 *   rope    — Alg. 2 l.379 rotary_pos_emb (rotate-half convention; reading R29), used
 *             only by the Eq. 5 block-level comparison (f4).
 *   attend  — Alg. 2 l.376-381 and Eq. 5:
 *             AttnMaps = softmax(Q K^T / sqrt(d_k)) with the causal mask of a
 *             decoder LLM (keys j <= i), then mat_mul(attn_map, v).
 *   project — Alg. 1 l.254 "f <- feature_projector(h)" with the
 *             projector of PAPER.md:278 ("two layers of Multi-Layer Perceptron
 *             ... maps the input embedding to a feature vector"): z = relu(W1 h
 *             + b1), y = W2 z + b2, f = y / ||y||_2 (readings R30-R32).
 *   linear  — Alg. 2 l.372, l.377-378 "v = V(h)", "q = Q(h)", "k = K(h)": the
 *             projections of the Eq. 5 block-level comparison (f4), Y = X W^T with W in the nn.Linear
 *             layout [N][K] (reading R34).
 *
 * Parity pins for each function live in tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Storage dtype codes understood by the oracle (its own numbering). */
enum { ORACLE_F32 = 0, ORACLE_F16 = 1, ORACLE_BF16 = 2 };

/* ---- exact decoders ---------------------------------------------------- */

static double dec_f32(uint32_t bits) {
    float f;
    memcpy(&f, &bits, 4);
    return (double)f;
}

/* bf16 is the top half of an IEEE binary32. */
static double dec_bf16(uint16_t h) { return dec_f32((uint32_t)h << 16); }

/* IEEE binary16: 1 sign, 5 exponent (bias 15), 10 mantissa bits. */
static double dec_f16(uint16_t h) {
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24); /* subnormal: m * 2^-14 * 2^-10 */
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = ldexp((double)(m | 0x400), e - 25); /* (1 + m/1024) * 2^(e-15) */
    return sign ? -v : v;
}

static double load(const void *base, int64_t i, int dtype) {
    switch (dtype) {
    case ORACLE_F32: return dec_f32(((const uint32_t *)base)[i]);
    case ORACLE_F16: return dec_f16(((const uint16_t *)base)[i]);
    default:         return dec_bf16(((const uint16_t *)base)[i]);
    }
}

double oracle_decode(const void *base, int64_t i, int32_t dtype) { return load(base, i, dtype); }

void oracle_set_threads(int32_t n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int32_t oracle_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- search: Alg. 1 l.255-257 ----------------------------------------- */

/* s = sum_k q[b][k] * x[i][k], in fp64. */
static double inner(const void *q, int64_t b, const void *x, int64_t i, int32_t D, int dtype) {
    double s = 0.0;
    for (int32_t k = 0; k < D; ++k)
        s += load(q, b * (int64_t)D + k, dtype) * load(x, i * (int64_t)D + k, dtype);
    return s;
}

/*
 * Brute-force top-1 for every query b in [0, B):
 *   idx[b] = the lowest i attaining max_i s[b][i]   (scan ascending, update on ">")
 *   s1[b]  = that maximum, s2[b] = the runner-up score (equal to s1 on a tie)
 *   hit[b] = s1[b] >= (double)tau                     (">=")
 * N == 0 gives idx = -1, s1 = s2 = -inf, hit = 0.
 */
void oracle_search(const void *q, int64_t B, const void *x, int64_t N, int32_t D, int32_t dtype,
                   float tau, int64_t *idx, double *s1, double *s2, uint8_t *hit) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b) {
        double best = -INFINITY, second = -INFINITY;
        int64_t arg = -1;
        for (int64_t i = 0; i < N; ++i) {
            double s = inner(q, b, x, i, D, dtype);
            if (s > best) {
                second = best;
                best = s;
                arg = i;
            } else if (s > second) {
                second = s;
            }
        }
        idx[b] = arg;
        s1[b] = best;
        s2[b] = second;
        hit[b] = (arg >= 0 && best >= (double)tau) ? 1 : 0;
    }
}

/* s[p] = q[qb[p]] . x[xi[p]] for a list of (query, entry) pairs. */
void oracle_scores(const void *q, const void *x, int32_t D, int32_t dtype, const int64_t *qb,
                   const int64_t *xi, int64_t n_pairs, double *s) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n_pairs; ++p) s[p] = inner(q, qb[p], x, xi[p], D, dtype);
}

/* ---- apply: Alg. 2 l.373-375, O = A . V -------------------------------- */

/*
 * One (query, layer, head) unit: A is [S][S] row-major (a_dtype), V is [S][d]
 * row-major (v_dtype); O[i][c] = sum_{j=0}^{S-1} A[i][j] * V[j][c].
 */
static void apply_unit(const void *A, int64_t a_off, int a_dtype, const void *V, int64_t v_off,
                       int v_dtype, int32_t S, int32_t d, double *O) {
    for (int32_t i = 0; i < S; ++i)
        for (int32_t c = 0; c < d; ++c) {
            double acc = 0.0;
            for (int32_t j = 0; j < S; ++j)
                acc += load(A, a_off + (int64_t)i * S + j, a_dtype) *
                       load(V, v_off + (int64_t)j * d + c, v_dtype);
            O[(int64_t)i * d + c] = acc;
        }
}

/* n_units independent units; unit u reads A at element offset a_off[u] and V at v_off[u],
 * and writes O + u*S*d. */
void oracle_apply(const void *A, int32_t a_dtype, const int64_t *a_off, const void *V, int32_t v_dtype,
                  const int64_t *v_off, int64_t n_units, int32_t S, int32_t d, double *O) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t u = 0; u < n_units; ++u)
        apply_unit(A, a_off[u], a_dtype, V, v_off[u], v_dtype, S, d, O + u * (int64_t)S * d);
}

/* ---- attend: Alg. 2 l.376-381, Eq. 5 ----------------------------------- */

/*
 * Causal attention probabilities of one unit: P[i][j] = exp(z_ij - m_i) / sum_{j'<=i} exp(z_ij' - m_i)
 * for j <= i and 0 for j > i, with z_ij = scale * sum_c Q[i][c] K[j][c] and m_i = max_{j<=i} z_ij.
 * (Eq. 5, plus the causal mask; subtracting m_i leaves softmax unchanged.)
 */
static void attention_map_unit(const void *Q, const void *K, int64_t off, int dtype, int32_t S, int32_t d,
                               double scale, double *P) {
    for (int32_t i = 0; i < S; ++i) {
        double *row = P + (int64_t)i * S;
        double m = -INFINITY;
        for (int32_t j = 0; j < S; ++j) {
            if (j > i) {
                row[j] = 0.0;
                continue;
            }
            double z = 0.0;
            for (int32_t c = 0; c < d; ++c)
                z += load(Q, off + (int64_t)i * d + c, dtype) * load(K, off + (int64_t)j * d + c, dtype);
            row[j] = z * scale;
            if (row[j] > m) m = row[j];
        }
        double sum = 0.0;
        for (int32_t j = 0; j <= i; ++j) {
            row[j] = exp(row[j] - m);
            sum += row[j];
        }
        for (int32_t j = 0; j <= i; ++j) row[j] /= sum;
    }
}

void oracle_attention_map(const void *Q, const void *K, int32_t dtype, const int64_t *off, int64_t n_units,
                          int32_t S, int32_t d, double scale, double *P) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t u = 0; u < n_units; ++u)
        attention_map_unit(Q, K, off[u], dtype, S, d, scale, P + u * (int64_t)S * S);
}

/* O = softmax(Q K^T * scale, causal) . V for n_units units; Q, K, V share the element offset off[u]. */
void oracle_attend(const void *Q, const void *K, const void *V, int32_t dtype, const int64_t *off,
                   int64_t n_units, int32_t S, int32_t d, double scale, double *O) {
#pragma omp parallel
    {
        double *P = (double *)malloc(sizeof(double) * (size_t)S * (size_t)S);
#pragma omp for schedule(dynamic, 1)
        for (int64_t u = 0; u < n_units; ++u) {
            attention_map_unit(Q, K, off[u], dtype, S, d, scale, P);
            double *Ou = O + u * (int64_t)S * d;
            for (int32_t i = 0; i < S; ++i)
                for (int32_t c = 0; c < d; ++c) {
                    double acc = 0.0;
                    for (int32_t j = 0; j <= i; ++j)
                        acc += P[(int64_t)i * S + j] * load(V, off[u] + (int64_t)j * d + c, dtype);
                    Ou[(int64_t)i * d + c] = acc;
                }
        }
        free(P);
    }
}

/* ---- RoPE (Alg. 2 l.379 "rotary_pos_emb(q, k)"; used by the Eq. 5 block-level
 * comparison).  Reading R29: the rotate-half convention of Llama-family
 * models: for i < d/2 the pair (x_i, x_{i+d/2}) at position p is rotated by the angle
 * p * base^(-2i/d).  Y = RoPE(X) for n_units units of [S][d], position p = row index. */
void oracle_rope(const void *X, int32_t dtype, int64_t n_units, int32_t S, int32_t d, double base, double *Y) {
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n_units; ++u)
        for (int32_t p = 0; p < S; ++p)
            for (int32_t i = 0; i < d / 2; ++i) {
                const int64_t row = (u * S + p) * (int64_t)d;
                const double theta = pow(base, -2.0 * i / d);
                const double c = cos(p * theta), s = sin(p * theta);
                const double x1 = load(X, row + i, dtype), x2 = load(X, row + i + d / 2, dtype);
                Y[row + i] = x1 * c - x2 * s;
                Y[row + i + d / 2] = x2 * c + x1 * s;
            }
}

/* ---- feature projector: Alg. 1 l.254, PAPER.md:278 ------------------------
 * Readings: R30 h is the sentence's input embedding vector [E]; R31 the two MLP layers
 * are affine maps with a ReLU between them (the paper names no activation); R32 the feature vector
 * is L2-normalised (the DB holds unit vectors, north_star; reading R2), and y = 0 gives f = 0.
 *   z[j] = max(0, sum_k W1[j][k] h[k] + b1[j])     j < Hd
 *   y[c] = sum_j W2[c][j] z[j] + b2[c]             c < D
 *   f[c] = y[c] / sqrt(sum_c y[c]^2)
 * h: [B][E], W1: [Hd][E], W2: [D][Hd] in `dtype`; b1: [Hd], b2: [D] fp32; f: [B][D] fp64. */
void oracle_project(const void *h, int64_t B, int32_t E, int32_t dtype, const void *W1, const float *b1,
                    int32_t Hd, const void *W2, const float *b2, int32_t D, double *f) {
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < B; ++b) {
        double *z = (double *)malloc(sizeof(double) * (size_t)(Hd > 0 ? Hd : 1));
        double *y = f + b * (int64_t)D;
        for (int32_t j = 0; j < Hd; ++j) {
            double s = 0.0;
            for (int32_t k = 0; k < E; ++k) s += load(W1, (int64_t)j * E + k, dtype) * load(h, b * (int64_t)E + k, dtype);
            s += (double)b1[j];
            z[j] = s > 0.0 ? s : 0.0;
        }
        double nn = 0.0;
        for (int32_t c = 0; c < D; ++c) {
            double s = 0.0;
            for (int32_t j = 0; j < Hd; ++j) s += load(W2, (int64_t)c * Hd + j, dtype) * z[j];
            y[c] = s + (double)b2[c];
            nn += y[c] * y[c];
        }
        const double norm = sqrt(nn);
        for (int32_t c = 0; c < D; ++c) y[c] = norm > 0.0 ? y[c] / norm : 0.0;
        free(z);
    }
}

/* ---- projections: Alg. 2 l.372, l.377-378 -------------
 * Y[m][n] = sum_k X[m][k] * W[n][k]: X [M][K], W [N][K] (the nn.Linear layout) in `dtype`; Y [M][N] fp64. */
void oracle_linear(const void *X, int64_t M, int32_t K, const void *W, int32_t N, int32_t dtype, double *Y) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m)
        for (int32_t n = 0; n < N; ++n) {
            double s = 0.0;
            for (int32_t k = 0; k < K; ++k) s += load(X, m * K + k, dtype) * load(W, (int64_t)n * K + k, dtype);
            Y[m * N + n] = s;
        }
}
