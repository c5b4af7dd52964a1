// item_sched.cuh — the work-item order shared by the persistent attention and capture kernels.
//
// A unit is one (selected row, layer, head) of a batch; an item is one 128-query block qb of a unit.  Items
// t = 0 .. units * n_qb - 1 are taken in L2-sized unit groups (the K/V of `group` units fit in about 48 MB
// of L2, so the re-reads of a unit's K/V blocks by its query blocks hit L2) and, inside a group, heaviest
// query block first (the persistent CTAs finish together).  The last group holds the batch's tail.
// All divisions by launch-time constants use host-made magics (FastDiv): the decode runs in every role
// of a CTA at every item switch, and plain 32-bit divisions put ~150 cycles on that path per item.
#pragma once
#include <algorithm>
#include <cstdint>

#include "sm100.cuh"

namespace ac {

struct ItemSched {
    uint32_t group, n_qb, per_row, S, L, Hkv;
    uint32_t rotate = 0;  // wave order (make_wave): query-block levels rotate by group index
    sm100::FastDiv gq, grp, per_row_d, h_d, hq_d, qb_d;  // group * n_qb, group, L * H, H, H / Hkv, n_qb

    // unit_bytes: L2 bytes one unit keeps live (its K and V, or K alone); blk: query block rows
    __host__ static ItemSched make(uint32_t S, uint32_t L, uint32_t H, uint32_t Hkv, uint32_t blk, uint32_t unit_bytes) {
        ItemSched c;
        c.S = S;
        c.n_qb = (S + blk - 1) / blk;  // a last, partial query block when S % blk != 0
        c.per_row = L * H;
        c.L = L;
        c.Hkv = Hkv;
        c.group = std::max(1u, (48u << 20) / unit_bytes);
        c.gq = sm100::FastDiv(c.group * c.n_qb);
        c.grp = sm100::FastDiv(c.group);
        c.per_row_d = sm100::FastDiv(c.per_row);
        c.h_d = sm100::FastDiv(H);
        c.hq_d = sm100::FastDiv(H / Hkv);
        c.qb_d = sm100::FastDiv(c.n_qb);
        return c;
    }

    // Wave order: a group holds as many items as there are item streams (one wave), so the streams work on
    // few units at a time (their K/V stay in L2 across the query blocks); the query-block level of a
    // stream's item rotates from group to group, so every stream gets every level in turn.
    __host__ static ItemSched make_wave(uint32_t S, uint32_t L, uint32_t H, uint32_t Hkv, uint32_t blk, uint32_t streams) {
        ItemSched c = make(S, L, H, Hkv, blk, 1u << 30);
        c.group = std::max(1u, streams / c.n_qb);
        c.gq = sm100::FastDiv(c.group * c.n_qb);
        c.grp = sm100::FastDiv(c.group);
        c.rotate = c.n_qb > 1 ? 1u : 0u;  // one query block per unit: the plain unit order
        return c;
    }

    struct Item {
        int64_t row0;     // first Q / O row of the unit ([rows][L][H][S] flattened) = unit * S
        int64_t kv_row0;  // first K / V row (grouped-query attention: K/V head h / (H / Hkv)) = kv_unit * S
        int32_t unit;     // the Q / O unit index ([rows][L][H]): the outer coordinate of the 3-D tensor maps
        int32_t kv_unit;  // the K / V unit index ([rows][L][Hkv])
        int64_t row;      // the selected batch row
        uint32_t lh;      // layer * H + head
        int qb;           // query block
    };

    __host__ __device__ __forceinline__ Item decode(uint32_t t, uint32_t units, const int32_t *rows) const {
        Item it;
        const uint32_t gi = gq.div(t), w = t - gi * gq.d;
        const uint32_t gbase = gi * group;
        uint32_t u;
        uint32_t a;
        if (gbase + group <= units) {
            a = grp.div(w);
            u = gbase + (w - a * group);
        } else {  // the last, partial group
            const uint32_t gsize = units - gbase;
            a = w / gsize;
            u = gbase + w % gsize;
        }
        if (rotate) a = qb_d.mod(a + qb_d.mod(gi));
        it.qb = (int)(n_qb - 1 - a);
        const uint32_t ri = per_row_d.div(u);
        it.lh = u - ri * per_row;
        it.row = rows[ri];
        const uint32_t l = h_d.div(it.lh), h = it.lh - l * h_d.d;
        it.unit = (int32_t)(it.row * per_row + it.lh);
        it.kv_unit = (int32_t)((it.row * L + l) * Hkv + hq_d.div(h));
        it.row0 = (int64_t)it.unit * S;
        it.kv_row0 = (int64_t)it.kv_unit * S;
        return it;
    }
};

// One CTA-local item stream: items first, first + stride, ...; j walks the current item's key blocks.
// The schedule is passed to every call (not stored) so that, called with the kernel's __grid_constant__
// parameter, its fields are read from the constant bank rather than through a generic pointer.
struct ItemWalker {
    uint32_t t, stride, items, units;
    const int32_t *rows;
    bool active = false;
    int64_t row0 = 0, kv_row0 = 0;
    int32_t unit = 0, kv_unit = 0;
    int qb = 0, j = 0;
    __device__ __forceinline__ void init(const ItemSched &sc, uint32_t first, uint32_t stride_, uint32_t items_,
                                         uint32_t units_, const int32_t *rows_) {
        t = first, stride = stride_, items = items_, units = units_, rows = rows_;
        start_item(sc);
    }
    __device__ __forceinline__ void start_item(const ItemSched &sc) {
        active = t < items;
        if (!active) return;
        const ItemSched::Item it = sc.decode(t, units, rows);
        row0 = it.row0;
        kv_row0 = it.kv_row0;
        unit = it.unit;
        kv_unit = it.kv_unit;
        qb = it.qb;
        j = 0;
    }
    // Moves past the current key block; returns true when that block ended the item.
    __device__ __forceinline__ bool advance(const ItemSched &sc) {
        if (++j > qb) {
            t += stride;
            start_item(sc);
            return true;
        }
        return false;
    }
};

}  // namespace ac
