// Host-side check (no GPU) of the persistent kernels' work-item order, item_sched.cuh, and of the division
// magics it uses (FastDiv, sm100.cuh).  Built with nvcc and run by tests/test_native_host.py.
//   * FastDiv(d).div(n) == n / d for every divisor 1..4096 against edge and random numerators, and for
//     random 32-bit divisors;
//   * ItemSched::decode over t = 0 .. units * n_qb - 1 visits every (unit, query block) exactly once, in
//     L2-sized unit groups, heaviest query block first inside a group, with row0 / kv_row0 equal to the
//     plain-division formulas (grouped-query attention included), for shapes whose unit count does and
//     does not divide into whole groups.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "item_sched.cuh"

using ac::ItemSched;
using ac::sm100::FastDiv;

static uint64_t rng = 0x9e3779b97f4a7c15ull;
static uint32_t next32() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return (uint32_t)(rng >> 16);
}

static int fail(const char *what, long long a, long long b, long long c) {
    std::printf("FAIL %s: %lld %lld %lld\n", what, a, b, c);
    return 1;
}

static int check_fastdiv() {
    for (uint32_t d = 1; d <= 4096; ++d) {
        const FastDiv f(d);
        const uint32_t edge[] = {0u, 1u, d - 1, d, d + 1, 2 * d - 1, 2 * d, 0x7fffffffu, 0x80000000u, 0xfffffffeu, 0xffffffffu};
        for (uint32_t n : edge)
            if (f.div(n) != n / d || f.mod(n) != n % d) return fail("fastdiv edge", d, n, f.div(n));
        for (int i = 0; i < 2000; ++i) {
            const uint32_t n = next32();
            if (f.div(n) != n / d) return fail("fastdiv random", d, n, f.div(n));
        }
    }
    for (int i = 0; i < 200000; ++i) {
        const uint32_t d = next32() | 1u, n = next32();
        if (FastDiv(d).div(n) != n / d) return fail("fastdiv 32-bit", d, n, FastDiv(d).div(n));
    }
    return 0;
}

// S, L, H, Hkv, n_rows, unit_bytes (wave: streams, for ItemSched::make_wave)
static int check_sched(uint32_t S, uint32_t L, uint32_t H, uint32_t Hkv, uint32_t n_rows, uint32_t unit_bytes,
                       uint32_t wave = 0) {
    const ItemSched sc = wave ? ItemSched::make_wave(S, L, H, Hkv, 128, wave) : ItemSched::make(S, L, H, Hkv, 128, unit_bytes);
    std::vector<int32_t> rows(n_rows);
    for (uint32_t i = 0; i < n_rows; ++i) rows[i] = (int32_t)(3 * i + 1);  // a selected-row list (distinct rows)
    const uint32_t units = n_rows * L * H, items = units * sc.n_qb;
    std::vector<int> seen((size_t)units * sc.n_qb, 0);
    int last_group = -1, last_qb = 1 << 30;
    for (uint32_t t = 0; t < items; ++t) {
        const ItemSched::Item it = sc.decode(t, units, rows.data());
        // the unit back from row0: row0 = (row * L*H + lh) * S
        const uint32_t ri = (uint32_t)(std::find(rows.begin(), rows.end(), (int32_t)it.row) - rows.begin());
        const uint32_t u = ri * L * H + it.lh;
        if (ri >= n_rows || u >= units || it.qb < 0 || it.qb >= (int)sc.n_qb) return fail("decode range", t, u, it.qb);
        if (sc.n_qb != (S + 127) / 128) return fail("n_qb", S, sc.n_qb, 0);
        if (it.row0 != ((int64_t)it.row * L * H + it.lh) * S) return fail("row0", t, it.row0, 0);
        if (it.unit != (int32_t)((int64_t)it.row * L * H + it.lh)) return fail("unit", t, it.unit, 0);
        const uint32_t l = it.lh / H, h = it.lh % H;
        if (it.kv_row0 != (((int64_t)it.row * L + l) * Hkv + h / (H / Hkv)) * (int64_t)S) return fail("kv_row0", t, it.kv_row0, 0);
        if ((int64_t)it.kv_unit * S != it.kv_row0) return fail("kv_unit", t, it.kv_unit, 0);
        if (seen[(size_t)u * sc.n_qb + it.qb]++) return fail("item twice", t, u, it.qb);
        const int g = (int)(u / sc.group);
        if (g != (int)(t / (sc.group * sc.n_qb))) return fail("group order", t, g, 0);
        if (g != last_group) {
            last_group = g;
            last_qb = 1 << 30;
        }
        if (!sc.rotate && it.qb > last_qb) return fail("heaviest first", t, it.qb, last_qb);
        last_qb = it.qb;
    }
    for (size_t i = 0; i < seen.size(); ++i)
        if (seen[i] != 1) return fail("item missing", (long long)i, seen[i], 0);
    return 0;
}

int main() {
    int bad = check_fastdiv();
    // configs[1]-[3] misses (attention: K and V live per unit; capture: K), a partial last group, GQA, S = 8192
    bad |= check_sched(128, 16, 32, 32, 51, 2 * 128 * 64 * 2);
    bad |= check_sched(256, 32, 32, 32, 13, 2 * 256 * 128 * 2);
    bad |= check_sched(1024, 8, 32, 32, 16, 2 * 1024 * 128 * 2);
    bad |= check_sched(1024, 8, 32, 32, 16, 1024 * 128 * 2);
    bad |= check_sched(384, 2, 8, 2, 7, 2 * 384 * 128 * 2);
    bad |= check_sched(8192, 1, 4, 1, 3, 2 * 8192 * 128 * 2);
    bad |= check_sched(256, 3, 6, 3, 5, 40u << 20);  // groups of one unit
    bad |= check_sched(1024, 8, 32, 32, 16, 0, 296);  // wave order (capture: two streams per CTA)
    bad |= check_sched(1024, 8, 32, 32, 16, 0, 148);
    bad |= check_sched(384, 2, 8, 2, 7, 0, 148);
    // S % 128 != 0: a last, partial query block (the paper's context lengths, Table 3: 373 / 1019 tokens)
    bad |= check_sched(200, 4, 8, 8, 5, 2 * 200 * 128 * 2);
    bad |= check_sched(373, 2, 8, 2, 3, 2 * 373 * 128 * 2);
    bad |= check_sched(1019, 2, 4, 4, 3, 0, 148);
    bad |= check_sched(40, 2, 4, 4, 3, 2 * 40 * 64 * 2);
    std::printf(bad ? "item_sched_check FAILED\n" : "item_sched_check ok\n");
    return bad;
}
