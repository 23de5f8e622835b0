// Viewshed ray template (decision D5) — product code.
//
// SPEC.md:288,322 leave the R2 cell rule open; the frozen rule is:
//   rays  = primitive directions of the midpoint-circle perimeter cells of
//           radius roi ("midpoint-circle rasterization") plus the
//           8 principal directions ("exact agreement on the 8
//           axis/diagonal rays"), in angle order starting at (0,+1);
//   owner = every lattice-disk cell (a,b) != (0,0) belongs to the forward ray
//           with least perpendicular distance, ties to the lowest ray index.
// Perpendicular distance |a q - b p| / |(p,q)| = |cell| * |sin(dtheta)| is
// monotone in the angle gap for forward rays, so the owner is one of the two
// rays bracketing the cell's angle: binary search + 2 exact int64 compares per
// cell instead of the O(cells x rays) scan the oracle uses.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <tuple>

#include "ctx.hpp"

namespace txs {

namespace {

struct Dir { int64_t p, q; };   // p = row offset, q = col offset

inline int half_plane(const Dir& d) { return (d.p > 0 || (d.p == 0 && d.q > 0)) ? 0 : 1; }
// strict angle order with x = q, y = p
inline bool angle_less(const Dir& a, const Dir& b) {
    const int ha = half_plane(a), hb = half_plane(b);
    if (ha != hb) return ha < hb;
    return a.q * b.p - a.p * b.q > 0;
}

std::vector<Dir> perimeter(int64_t R) {
    std::vector<Dir> v;
    int64_t x = R, y = 0, err = 1 - R;
    while (x >= y) {
        v.push_back({x, y});   v.push_back({y, x});
        v.push_back({-y, x});  v.push_back({-x, y});
        v.push_back({-x, -y}); v.push_back({-y, -x});
        v.push_back({y, -x});  v.push_back({x, -y});
        ++y;
        if (err < 0) err += 2 * y + 1;
        else { --x; err += 2 * (y - x) + 1; }
    }
    return v;
}

RayTemplate build(int32_t R) {
    RayTemplate T;
    T.roi = R;
    std::vector<Dir> dirs;
    for (const Dir& d : perimeter(R)) {
        const int64_t g = std::gcd(std::llabs(d.p), std::llabs(d.q));
        dirs.push_back({d.p / g, d.q / g});
    }
    for (int64_t p = -1; p <= 1; ++p)
        for (int64_t q = -1; q <= 1; ++q)
            if (p || q) dirs.push_back({p, q});
    std::sort(dirs.begin(), dirs.end(), angle_less);
    dirs.erase(std::unique(dirs.begin(), dirs.end(),
                           [](const Dir& a, const Dir& b) { return a.p == b.p && a.q == b.q; }),
               dirs.end());
    const int64_t n = (int64_t)dirs.size();
    for (const Dir& d : dirs) { T.p.push_back((int32_t)d.p); T.q.push_back((int32_t)d.q); }

    std::vector<std::vector<std::tuple<int64_t, int32_t, int32_t>>> own((size_t)n);
    for (int64_t a = -R; a <= R; ++a)
        for (int64_t b = -R; b <= R; ++b) {
            if ((a == 0 && b == 0) || a * a + b * b > (int64_t)R * R) continue;
            const Dir c{a, b};
            // first ray not less than the cell's direction
            const int64_t hi = std::lower_bound(dirs.begin(), dirs.end(), c, angle_less) - dirs.begin();
            const int64_t r1 = hi % n, r0 = (hi + n - 1) % n;
            auto key = [&](int64_t r, int64_t* c2, int64_t* l2) {
                const int64_t cr = a * dirs[r].q - b * dirs[r].p;
                *c2 = cr * cr;
                *l2 = dirs[r].p * dirs[r].p + dirs[r].q * dirs[r].q;
            };
            int64_t c0, l0, c1, l1;
            key(r0, &c0, &l0);
            key(r1, &c1, &l1);
            int64_t best;
            const __int128 lhs = (__int128)c1 * l0, rhs = (__int128)c0 * l1;   // c1/l1 vs c0/l0
            if (lhs < rhs) best = r1;
            else if (lhs > rhs) best = r0;
            else best = std::min(r0, r1);
            own[(size_t)best].emplace_back(a * dirs[best].p + b * dirs[best].q, (int32_t)a, (int32_t)b);
        }
    T.cell_begin.push_back(0);
    for (int64_t r = 0; r < n; ++r) {
        std::sort(own[(size_t)r].begin(), own[(size_t)r].end());
        for (auto& [d, a, b] : own[(size_t)r]) { T.ca.push_back(a); T.cb.push_back(b); }
        T.cell_begin.push_back((int64_t)T.ca.size());
    }
    return T;
}

// Merged per-ray event stream (decision D5 evaluated in u order): for each ray
// the crossings of its primitive direction interleaved with its owned cells,
// a cell emitted before every crossing with u_k >= u_c, nothing after the
// last cell.  Event (uint2):
//   x: bits 0-2 type, 3-11 row offset dr (9-bit two's complement) of the
//      crossing's FIRST interpolation post, 12-21 F = 2*dc + (column crossing)
//      (10-bit two's complement; dc = F >> 1, and F is the word offset of the
//      post's pair in the interleaved (H, V) pair planes), 24-31 its weight w0
//      (so that one byte permute yields the dp2a weight word);
//   y: bits 0-23 the crossing's line index (its slope's M) or, for a cell, its
//      projection numerator dot = a*p + b*q; bits 24-31 the weight w1 of the
//      second post, which lies one column right (row crossing) or one row down
//      (column crossing) of the first.
// The interpolated height times the crossing's denominator n is
// z0*w0 + z1*w1 with w0 + w1 = n (the pair is ordered by increasing column /
// row whatever the ray's direction, so the GPU can read it as one packed pair);
// posts carry (n, 0), cells (1, 0).
inline uint2 pack_ev(uint32_t type, int dr, int dc, int w0, int w1, int64_t y) {
    // bits 12..21 hold 2*dc + (column crossing): the word offset of the crossing's
    // pair in the interleaved (H, V) pair planes, one IMAD from dr (viewshed.cu)
    const uint32_t f = (uint32_t)(2 * dc + (type == kEvCol ? 1 : 0)) & 0x3ffu;
    return make_uint2(type | ((uint32_t)(dr & 0x1ff) << 3) | (f << 12) | ((uint32_t)w0 << 24),
                      (uint32_t)y | ((uint32_t)w1 << 24));
}

// Interior-sweep encoding of the same event (k_viewshed_evk's interior
// observers share the window pitch 2R+1, so a cell's bitmap bit is a template
// constant):
//   x: bits 0-1 type (kEv3Cross / kEv3Cell / kEv3Nop), 2-10 dr, 11-20 F =
//      2*dc + (column crossing) (two's complement; the pair offset is
//      dr*p2 + F), 21-31 aux bits 0-10;
//   y: bits 0-24 yv, 25-31 aux bits 11-17.
// crossing: aux = w0 | w1 << 8 (the dp2a weight word), yv = line index * L2
//   (the horizon then keeps M' = L2*M, so cells and crossings share one
//   product X*M' and no select); cell: aux = its bit in the interior window
//   bitmap, (dr + R)*(2R+1) + dc + R, yv = dot.  Bounds (R <= 250): line
//   index * L2 <= 2R^3 < 2^25, bit index < (2R+1)^2 < 2^18.
inline uint2 pack_ev3(uint2 e, int64_t R, int64_t L2) {
    const uint32_t t2 = e.x & 7u;
    const int dr = ((int)(e.x << 20)) >> 23, F = ((int)(e.x << 10)) >> 22, dc = F >> 1;
    uint32_t type, aux;
    uint64_t yv;
    if (t2 == kEvNop) return make_uint2(kEv3Nop, 0u);
    if (t2 == kEvCell) {
        type = kEv3Cell;
        aux = (uint32_t)((dr + R) * (2 * R + 1) + dc + R);
        yv = e.y & 0xffffffu;
    } else {
        type = kEv3Cross;
        aux = (e.x >> 24) | ((e.y >> 24) << 8);
        yv = (uint64_t)(e.y & 0xffffffu) * (uint64_t)L2;
    }
    if (yv >= (1u << 25) || aux >= (1u << 18)) throw std::runtime_error("event3 field overflow");
    return make_uint2(type | ((uint32_t)(dr & 0x1ff) << 2) | ((uint32_t)(F & 0x3ff) << 11) | ((aux & 0x7ffu) << 21),
                      (uint32_t)yv | ((aux >> 11) << 25));
}

EventTemplate build_events(const RayTemplate& T) {
    EventTemplate E;
    const int64_t nrays = (int64_t)T.p.size();
    std::vector<std::vector<uint2>> per((size_t)nrays);
    for (int64_t r = 0; r < nrays; ++r) {
        const int64_t p = T.p[(size_t)r], q = T.q[(size_t)r];
        const int64_t ap = std::llabs(p), aq = std::llabs(q), sp = p >= 0 ? 1 : -1, sq = q >= 0 ? 1 : -1;
        const int64_t L2 = p * p + q * q;
        const int64_t dqr = ap ? aq / ap : 0, dmr = ap ? aq % ap : 0, dqc = aq ? ap / aq : 0, dmc = aq ? ap % aq : 0;
        int64_t i = 1, j = 1, qr = dqr, mr = dmr, qc = dqc, mc = dmc;
        auto& ev = per[(size_t)r];
        for (int64_t k = T.cell_begin[(size_t)r]; k < T.cell_begin[(size_t)r + 1]; ++k) {
            const int64_t a = T.ca[(size_t)k], b = T.cb[(size_t)k], dot = a * p + b * q;
            for (;;) {
                bool isrow, iscol;
                if (ap == 0) { isrow = false; iscol = true; }
                else if (aq == 0) { isrow = true; iscol = false; }
                else { const int64_t cmp = i * aq - j * ap; isrow = cmp <= 0; iscol = cmp >= 0; }
                const int64_t idx = isrow ? i : j, n = isrow ? ap : aq;
                if (idx * L2 >= dot * n) break;
                if (isrow && iscol) {
                    ev.push_back(pack_ev(kEvPost, (int)(sp * i), (int)(sq * j), (int)ap, 0, i));
                } else if (isrow) {   // posts (sp*i, sq*qr) weight ap-mr and (sp*i, sq*qr+sq) weight mr
                    if (aq == 0) ev.push_back(pack_ev(kEvPost, (int)(sp * i), 0, (int)ap, 0, i));
                    else if (sq > 0) ev.push_back(pack_ev(kEvRow, (int)(sp * i), (int)qr, (int)(ap - mr), (int)mr, i));
                    else ev.push_back(pack_ev(kEvRow, (int)(sp * i), (int)(-qr - 1), (int)mr, (int)(ap - mr), i));
                } else {              // posts (sp*qc, sq*j) weight aq-mc and (sp*qc+sp, sq*j) weight mc
                    if (ap == 0) ev.push_back(pack_ev(kEvPost, 0, (int)(sq * j), (int)aq, 0, j));
                    else if (sp > 0) ev.push_back(pack_ev(kEvCol, (int)qc, (int)(sq * j), (int)(aq - mc), (int)mc, j));
                    else ev.push_back(pack_ev(kEvCol, (int)(-qc - 1), (int)(sq * j), (int)mc, (int)(aq - mc), j));
                }
                if (isrow) { ++i; qr += dqr; mr += dmr; if (mr >= ap) { mr -= ap; ++qr; } }
                if (iscol) { ++j; qc += dqc; mc += dmc; if (mc >= aq) { mc -= aq; ++qc; } }
            }
            ev.push_back(pack_ev(kEvCell, (int)a, (int)b, 1, 0, dot));
        }
    }
    const int64_t ngroups = (nrays + 31) / 32;
    int64_t row = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
        size_t steps = 0;
        for (int64_t l = 0; l < 32 && g * 32 + l < nrays; ++l) steps = std::max(steps, per[(size_t)(g * 32 + l)].size());
        steps = (steps + 3) & ~(size_t)3;   // a multiple of 4: the sweeps read 2 or 4 steps per iteration without a bound test
        E.groups.push_back(make_int2((int)row, (int)steps));
        for (size_t s = 0; s < steps; ++s)
            for (int64_t l = 0; l < 32; ++l) {
                const int64_t r = g * 32 + l;
                const uint2 e = r < nrays && s < per[(size_t)r].size() ? per[(size_t)r][s]
                                                                       : make_uint2((uint32_t)kEvNop, 0u);
                E.events.push_back(e);
                const int64_t L2 = r < nrays ? (int64_t)T.p[(size_t)r] * T.p[(size_t)r] +
                                                   (int64_t)T.q[(size_t)r] * T.q[(size_t)r] : 1;
                E.events3.push_back(pack_ev3(e, T.roi, L2));
            }
        row += (int64_t)steps;
    }
    // 4 rows of Nops past the last group: the sweeps prefetch one iteration ahead
    for (int s = 0; s < 4 * 32; ++s) {
        E.events.push_back(make_uint2((uint32_t)kEvNop, 0u));
        E.events3.push_back(make_uint2((uint32_t)kEv3Nop, 0u));
    }
    return E;
}

}  // namespace

const EventTemplate& event_template(int32_t roi) {
    static std::mutex mu;
    static std::map<int32_t, EventTemplate> cache;
    const RayTemplate& T = ray_template(roi);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(roi);
    if (it == cache.end()) it = cache.emplace(roi, build_events(T)).first;
    return it->second;
}

const RayTemplate& ray_template(int32_t roi) {
    static std::mutex mu;
    static std::map<int32_t, RayTemplate> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(roi);
    if (it == cache.end()) it = cache.emplace(roi, build(roi)).first;
    return it->second;
}

txs_status get_template(txs_ctx* ctx, int32_t roi, RayTemplateDev** out) {
    auto it = ctx->templates.find(roi);
    if (it != ctx->templates.end()) { *out = &it->second; return TXS_OK; }
    const RayTemplate& T = ray_template(roi);
    RayTemplateDev D;
    D.roi = roi;
    D.nrays = (int32_t)T.p.size();
    D.ncells = (int64_t)T.ca.size();
    std::vector<int4> rays((size_t)D.nrays);
    for (int32_t r = 0; r < D.nrays; ++r)
        rays[(size_t)r] = make_int4(T.p[(size_t)r], T.q[(size_t)r], (int)T.cell_begin[(size_t)r],
                                    (int)(T.cell_begin[(size_t)r + 1] - T.cell_begin[(size_t)r]));
    std::vector<uint32_t> cells((size_t)D.ncells);
    for (int64_t i = 0; i < D.ncells; ++i)
        cells[(size_t)i] = ((uint32_t)(uint16_t)(int16_t)T.ca[(size_t)i]) |
                           ((uint32_t)(uint16_t)(int16_t)T.cb[(size_t)i] << 16);
    if (roi <= kEvMaxRoi) {
        const EventTemplate& E = event_template(roi);
        D.ngroups = (int32_t)E.groups.size();
        D.nevents = (int64_t)E.events.size();
        TXS_CUDA(ctx, "viewshed", cudaMalloc(&D.groups, sizeof(int2) * E.groups.size()));
        TXS_CUDA(ctx, "viewshed", cudaMalloc(&D.events, sizeof(uint2) * std::max<size_t>(1, E.events.size())));
        TXS_CUDA(ctx, "viewshed", cudaMalloc(&D.events3, sizeof(uint2) * std::max<size_t>(1, E.events3.size())));
        TXS_CUDA(ctx, "viewshed", cudaMemcpy(D.groups, E.groups.data(), sizeof(int2) * E.groups.size(), cudaMemcpyHostToDevice));
        if (!E.events.empty())
            TXS_CUDA(ctx, "viewshed", cudaMemcpy(D.events, E.events.data(), sizeof(uint2) * E.events.size(), cudaMemcpyHostToDevice));
        if (!E.events3.empty())
            TXS_CUDA(ctx, "viewshed", cudaMemcpy(D.events3, E.events3.data(), sizeof(uint2) * E.events3.size(), cudaMemcpyHostToDevice));
    }
    TXS_CUDA(ctx, "viewshed", cudaMalloc(&D.rays, sizeof(int4) * rays.size()));
    TXS_CUDA(ctx, "viewshed", cudaMalloc(&D.cells, sizeof(uint32_t) * std::max<size_t>(1, cells.size())));
    TXS_CUDA(ctx, "viewshed", cudaMemcpy(D.rays, rays.data(), sizeof(int4) * rays.size(), cudaMemcpyHostToDevice));
    if (!cells.empty())
        TXS_CUDA(ctx, "viewshed", cudaMemcpy(D.cells, cells.data(), sizeof(uint32_t) * cells.size(), cudaMemcpyHostToDevice));
    *out = &(ctx->templates[roi] = D);
    return TXS_OK;
}

}  // namespace txs

extern "C" int64_t txs_ray_template(int32_t roi, int32_t* p, int32_t* q, int64_t* cell_begin,
                                    int32_t* ca, int32_t* cb, int64_t cap_rays, int64_t cap_cells,
                                    int64_t* ncells) {
    if (roi < 1 || roi > 4000) return -1;
    const txs::RayTemplate& T = txs::ray_template(roi);
    const int64_t nr = (int64_t)T.p.size(), nc = (int64_t)T.ca.size();
    if (ncells) *ncells = nc;
    if (cap_rays >= nr && cap_cells >= nc && p && q && cell_begin && ca && cb) {
        std::copy(T.p.begin(), T.p.end(), p);
        std::copy(T.q.begin(), T.q.end(), q);
        std::copy(T.cell_begin.begin(), T.cell_begin.end(), cell_begin);
        std::copy(T.ca.begin(), T.ca.end(), ca);
        std::copy(T.cb.begin(), T.cb.end(), cb);
    }
    return nr;
}

extern "C" int txs_event_template_info(int32_t roi, int64_t* real_events, int64_t* padded_events, int32_t* groups) {
    if (roi < 1 || roi > txs::kEvMaxRoi || !real_events || !padded_events || !groups) return 1;
    const txs::EventTemplate& E = txs::event_template(roi);
    int64_t real = 0;
    for (const uint2& e : E.events) real += (e.x & 7u) != txs::kEvNop;
    *real_events = real;
    *padded_events = (int64_t)E.events.size();
    *groups = (int32_t)E.groups.size();
    return 0;
}
