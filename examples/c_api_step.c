/* c_api_step.c — the AttnCache step through the C ABI alone (include/attncache.h), no Python: a tiny database is
 * built on the device (its maps captured by attncache_capture_maps from random Q, K), then one batch is searched
 * (Alg. 1 l.255-257), the hits apply their cached maps (Alg. 2 l.373-375) and the misses run causal attention
 * (Alg. 2 l.376-381).  Checks: planted queries hit their entries, a random query misses, a hit's O equals the
 * attention of its entry's (Q, K) with its own V up to map rounding, every status is OK.  Exit code 0 = pass.
 *
 *   gcc -O2 -std=c11 -I include -I /usr/local/cuda/include examples/c_api_step.c \
 *       -L paper_2510_25979_b200/lib -lattncache -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,paper_2510_25979_b200/lib -o /tmp/c_api_step && /tmp/c_api_step
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "attncache.h"

#define CHECK(call)                                                                                   \
    do {                                                                                              \
        attncache_status s_ = (call);                                                                 \
        if (s_ != ATTNCACHE_OK) {                                                                     \
            fprintf(stderr, "%s:%d %s -> %s: %s\n", __FILE__, __LINE__, #call, attncache_status_string(s_), \
                    attncache_last_error());                                                          \
            return 1;                                                                                 \
        }                                                                                             \
    } while (0)
#define CUDA(call)                                                                                    \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) {                                                                      \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_));   \
            return 1;                                                                                 \
        }                                                                                             \
    } while (0)

enum { N = 4, L = 2, H = 2, S = 128, D_HEAD = 64, FEAT = 128, B = 3 };

static uint16_t to_bf16(float f) { /* round to nearest even */
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static float frand(unsigned *state) { /* a small LCG in [-1, 1) */
    *state = *state * 1664525u + 1013904223u;
    return ((*state >> 8) & 0xFFFFFF) / 8388608.0f - 1.0f;
}
static void *upload_bf16(const float *x, size_t n) {
    uint16_t *h = (uint16_t *)malloc(n * 2);
    for (size_t i = 0; i < n; ++i) h[i] = to_bf16(x[i]);
    void *d = NULL;
    if (cudaMalloc(&d, n * 2) != cudaSuccess) return NULL;
    cudaMemcpy(d, h, n * 2, cudaMemcpyHostToDevice);
    free(h);
    return d;
}

int main(void) {
    unsigned rng = 12345u;
    const size_t unit = (size_t)S * D_HEAD, act_n = (size_t)L * H * unit;
    /* database: N entries; features L2-normalised, maps captured from random (Q, K) of each entry */
    float *feat = (float *)malloc(sizeof(float) * N * FEAT);
    for (int i = 0; i < N; ++i) {
        double nrm = 0;
        for (int k = 0; k < FEAT; ++k) {
            feat[i * FEAT + k] = frand(&rng);
            nrm += feat[i * FEAT + k] * feat[i * FEAT + k];
        }
        for (int k = 0; k < FEAT; ++k) feat[i * FEAT + k] /= (float)sqrt(nrm);
    }
    float *qk = (float *)malloc(sizeof(float) * N * act_n);
    for (size_t i = 0; i < N * act_n; ++i) qk[i] = frand(&rng);
    void *d_feat = upload_bf16(feat, (size_t)N * FEAT);
    void *d_Qdb = upload_bf16(qk, N * act_n);
    for (size_t i = 0; i < N * act_n; ++i) qk[i] = frand(&rng);
    void *d_Kdb = upload_bf16(qk, N * act_n);
    if (!d_feat || !d_Qdb || !d_Kdb) return 1;

    attncache_ctx *ctx = NULL;
    CHECK(attncache_ctx_create(0, 0, 1, NULL, &ctx));
    const int64_t map_elems = attncache_packed_map_elems(S);
    void *d_maps = NULL;
    CUDA(cudaMalloc(&d_maps, (size_t)N * L * H * map_elems * 2));
    CHECK(attncache_capture_maps(ctx, N, L, H, S, D_HEAD, ATTNCACHE_BF16, d_Qdb, d_Kdb, 0.0f, NULL, ATTNCACHE_BF16,
                                 ATTNCACHE_MAPS_PACKED, d_maps, NULL));
    attncache_db_desc desc;
    memset(&desc, 0, sizeof desc);
    desc.n_global = N;
    desc.shard_begin = 0;
    desc.shard_count = N;
    desc.feat_dim = FEAT;
    desc.feat_dtype = ATTNCACHE_BF16;
    desc.feats = d_feat;
    desc.n_layers = L;
    desc.n_heads = H;
    desc.seq_len = S;
    desc.map_dtype = ATTNCACHE_BF16;
    desc.maps = d_maps;
    desc.map_layout = ATTNCACHE_MAPS_PACKED;
    attncache_db *db = NULL;
    CHECK(attncache_db_load(ctx, &desc, &db));

    /* batch: query 0 = entry 2 exactly, query 1 = entry 0 exactly, query 2 random (a miss at tau = 0.9) */
    float *q = (float *)malloc(sizeof(float) * B * FEAT);
    memcpy(q, feat + 2 * FEAT, sizeof(float) * FEAT);
    memcpy(q + FEAT, feat, sizeof(float) * FEAT);
    for (int k = 0; k < FEAT; ++k) q[2 * FEAT + k] = frand(&rng) / (float)sqrt((double)FEAT);
    void *d_q = upload_bf16(q, (size_t)B * FEAT);
    /* activations: V random; Q, K of row b = the Q, K of its planted entry (rows 0, 1), random for row 2 */
    float *v = (float *)malloc(sizeof(float) * B * act_n);
    for (size_t i = 0; i < B * act_n; ++i) v[i] = frand(&rng);
    void *d_V = upload_bf16(v, B * act_n);
    void *d_Q = NULL, *d_K = NULL, *d_O = NULL, *d_O2 = NULL;
    CUDA(cudaMalloc(&d_Q, B * act_n * 2));
    CUDA(cudaMalloc(&d_K, B * act_n * 2));
    CUDA(cudaMalloc(&d_O, B * act_n * 2));
    CUDA(cudaMalloc(&d_O2, B * act_n * 2));
    const int planted[2] = {2, 0};
    for (int b = 0; b < 2; ++b) {
        CUDA(cudaMemcpy((char *)d_Q + b * act_n * 2, (char *)d_Qdb + planted[b] * act_n * 2, act_n * 2, cudaMemcpyDeviceToDevice));
        CUDA(cudaMemcpy((char *)d_K + b * act_n * 2, (char *)d_Kdb + planted[b] * act_n * 2, act_n * 2, cudaMemcpyDeviceToDevice));
    }
    CUDA(cudaMemcpy((char *)d_Q + 2 * act_n * 2, d_V, act_n * 2, cudaMemcpyDeviceToDevice));
    CUDA(cudaMemcpy((char *)d_K + 2 * act_n * 2, (char *)d_V + act_n * 2, act_n * 2, cudaMemcpyDeviceToDevice));
    int64_t *d_idx = NULL;
    float *d_score = NULL;
    uint8_t *d_hit = NULL;
    CUDA(cudaMalloc((void **)&d_idx, B * sizeof(int64_t)));
    CUDA(cudaMalloc((void **)&d_score, B * sizeof(float)));
    CUDA(cudaMalloc((void **)&d_hit, B));

    /* the step: search, A.V for the hits, attention for the misses (skip = hit) */
    CHECK(attncache_search(db, d_q, B, 0.9f, d_idx, d_score, d_hit, NULL));
    CHECK(attncache_apply_cached(db, d_idx, d_hit, B, 0, L, D_HEAD, ATTNCACHE_BF16, d_V, d_O, NULL));
    CHECK(attncache_attend_full(ctx, B, L, H, S, D_HEAD, ATTNCACHE_BF16, d_Q, d_K, d_V, 0.0f, d_hit, d_O, NULL));
    /* reference for the hits: full attention of every row */
    CHECK(attncache_attend_full(ctx, B, L, H, S, D_HEAD, ATTNCACHE_BF16, d_Q, d_K, d_V, 0.0f, NULL, d_O2, NULL));
    CHECK(attncache_ctx_sync(ctx));

    int64_t idx[B];
    float score[B];
    uint8_t hit[B];
    CUDA(cudaMemcpy(idx, d_idx, sizeof idx, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(score, d_score, sizeof score, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(hit, d_hit, sizeof hit, cudaMemcpyDeviceToHost));
    int bad = 0;
    if (!(hit[0] && idx[0] == 2 && hit[1] && idx[1] == 0 && !hit[2])) {
        fprintf(stderr, "decisions: idx %lld %lld %lld hit %d %d %d\n", (long long)idx[0], (long long)idx[1],
                (long long)idx[2], hit[0], hit[1], hit[2]);
        bad = 1;
    }
    uint16_t *O = (uint16_t *)malloc(B * act_n * 2), *O2 = (uint16_t *)malloc(B * act_n * 2);
    CUDA(cudaMemcpy(O, d_O, B * act_n * 2, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(O2, d_O2, B * act_n * 2, cudaMemcpyDeviceToHost));
    double max_diff = 0;
    for (size_t i = 0; i < B * act_n; ++i) {
        const double dd = fabs((double)from_bf16(O[i]) - (double)from_bf16(O2[i]));
        if (dd > max_diff) max_diff = dd;
    }
    /* hits: A.V with the captured (bf16-rounded) maps vs attention on the same (Q, K, V); misses: identical */
    if (!(max_diff < 3e-2)) {
        fprintf(stderr, "cached vs full attention: max |diff| %g\n", max_diff);
        bad = 1;
    }
    printf("c_api_step: idx %lld %lld %lld, hit %d %d %d, score %.4f %.4f %.4f, max |O - O_full| %.2e: %s\n",
           (long long)idx[0], (long long)idx[1], (long long)idx[2], hit[0], hit[1], hit[2], score[0], score[1],
           score[2], max_diff, bad ? "FAIL" : "ok");
    CHECK(attncache_db_free(db));
    CHECK(attncache_ctx_destroy(ctx));
    return bad;
}
