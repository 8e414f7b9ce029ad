// Host-side sequential two-level cache planner.
//
// Exact re-implementation (not a translation: dense per-key tables, an
// intrusive order list and an ordered (score, key) set replace the Python
// dict + lazy heap) of halopart's CacheSystem (src/halopart/cache.py:137-347)
// and of simulator.run's round-robin lookup loop (simulator.py:206-226).
// It runs the transient epochs (before JACA membership freezes), every
// epoch of FIFO/LRU, and the replay when the GPU planner (K6) flags an
// admission.  Output tables drive the K3 staging / write-through kernels.

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/capgnn.h"

extern void cg_set_error(const std::string &msg);

namespace {

enum { POL_JACA = 0, POL_FIFO = 1, POL_LRU = 2 };
enum { OUT_LOCAL = 0, OUT_GLOBAL = 1, OUT_MISS = 2 };

struct Level {
    int policy = 0;
    int64_t capacity = 0;
    int64_t count = 0;
    // per key: slot (-1 absent), version, order links
    std::vector<int32_t> slot, ver, prev, next;
    int32_t head = -1, tail = -1;      // order list: head = oldest / LRU
    std::vector<int32_t> slot_key;     // slot -> key (-1 free)
    std::vector<uint8_t> slot_dirty;   // content changed in current epoch
    int64_t next_free = 0;
    std::set<std::pair<double, int32_t>> by_score;
    const std::vector<double> *score = nullptr;
    int64_t admissions = 0;

    void init(int pol, int64_t cap, int64_t n_keys, const std::vector<double> *sc) {
        policy = pol;
        capacity = cap;
        score = sc;
        slot.assign(n_keys, -1);
        ver.assign(n_keys, 0);
        prev.assign(n_keys, -1);
        next.assign(n_keys, -1);
        slot_key.assign(cap, -1);
        slot_dirty.assign(cap, 0);
    }
    bool has(int32_t k) const { return slot[k] >= 0; }
    double sc(int32_t k) const { return (*score)[k]; }
    void unlink(int32_t k) {
        int32_t p = prev[k], n = next[k];
        if (p >= 0) next[p] = n; else head = n;
        if (n >= 0) prev[n] = p; else tail = p;
        prev[k] = next[k] = -1;
    }
    void push_back(int32_t k) {
        prev[k] = tail;
        next[k] = -1;
        if (tail >= 0) next[tail] = k; else head = k;
        tail = k;
    }
    void touch(int32_t k) {
        if (policy == POL_LRU && has(k)) { unlink(k); push_back(k); }
    }
    void refresh(int32_t k, int32_t v) {
        ver[k] = v;
        slot_dirty[slot[k]] = 1;
        touch(k);
    }
    // returns evicted key or -1; rejected candidates leave the level intact
    int32_t insert(int32_t k, int32_t v) {
        if (has(k)) { refresh(k, v); return -1; }
        if (capacity == 0) return -1;
        int32_t victim = -1, s;
        if (count >= capacity) {
            if (policy == POL_JACA) {
                auto lo = by_score.begin();
                if (sc(k) <= lo->first) return -1;
                victim = lo->second;
                by_score.erase(lo);
            } else {
                victim = head;
            }
            s = slot[victim];
            unlink(victim);
            slot[victim] = -1;
            --count;
        } else {
            s = (int32_t)next_free++;
        }
        slot[k] = s;
        ver[k] = v;
        slot_key[s] = k;
        slot_dirty[s] = 1;
        push_back(k);
        if (policy == POL_JACA) by_score.insert({sc(k), k});
        ++count;
        ++admissions;
        return victim;
    }
    bool can_admit() const { return capacity > 0 && count < capacity; }
    // admit mode for a non-resident candidate: 0 never, 1 always, 2 iff its
    // score strictly beats the resident minimum (JACA on a full level)
    int admit_mode() const {
        if (capacity == 0) return 0;
        if (count < capacity || policy != POL_JACA) return 1;
        return 2;
    }
    double min_score() const { return by_score.empty() ? 0.0 : by_score.begin()->first; }
};

inline bool fresh(int32_t ver, int epoch, int s) { return s < 0 || epoch - ver <= s; }

}  // namespace

struct cg_planner {
    int policy = 0;
    int P = 0;
    int64_t n_keys = 0;
    std::vector<double> score;
    std::vector<Level> loc;
    Level glo;
    std::vector<int64_t> halo_off;
    std::vector<int32_t> halo, ranked;
    std::vector<int64_t> lookups, lh, gh, ms;
    std::vector<int64_t> lslot_off;

    // returns outcome and served version
    int lookup(int d, int32_t k, int e, int s, int32_t *served, int32_t *hit_slot) {
        Level &L = loc[d];
        ++lookups[d];
        bool lres = L.has(k);
        if (lres && fresh(L.ver[k], e, s)) {
            L.touch(k);
            ++lh[d];
            *served = L.ver[k];
            *hit_slot = L.slot[k];
            return OUT_LOCAL;
        }
        *hit_slot = -1;
        bool gres = glo.has(k);
        if (gres && fresh(glo.ver[k], e, s)) {
            glo.touch(k);
            int32_t gv = glo.ver[k];
            if (lres) L.refresh(k, gv); else L.insert(k, gv);
            ++gh[d];
            *served = gv;
            return OUT_GLOBAL;
        }
        if (gres) glo.refresh(k, e); else glo.insert(k, e);
        if (lres) L.refresh(k, e); else L.insert(k, e);
        ++ms[d];
        *served = e;
        return OUT_MISS;
    }
};

extern "C" {

int cg_planner_create(int policy, int n_parts, int64_t c_cpu, const int64_t *c_gpu,
                      int64_t n_union, const double *score, cg_planner **out) {
    if (policy < 0 || policy > 2 || n_parts < 1 || c_cpu < 0 || n_union < 0 || !out) {
        cg_set_error("cg_planner_create: bad arguments");
        return -1;
    }
    auto *p = new cg_planner();
    p->policy = policy;
    p->P = n_parts;
    p->n_keys = n_union;
    p->score.assign(score, score + n_union);
    p->loc.resize(n_parts);
    p->lslot_off.assign(n_parts + 1, 0);
    for (int d = 0; d < n_parts; ++d) {
        if (c_gpu[d] < 0) { delete p; cg_set_error("negative capacity"); return -1; }
        p->loc[d].init(policy, c_gpu[d], n_union, &p->score);
        p->lslot_off[d + 1] = p->lslot_off[d] + c_gpu[d];
    }
    p->glo.init(policy, c_cpu, n_union, &p->score);
    p->lookups.assign(n_parts, 0);
    p->lh = p->gh = p->ms = p->lookups;
    *out = p;
    return 0;
}

int cg_planner_destroy(cg_planner *p) {
    delete p;
    return 0;
}

int cg_planner_set_halos(cg_planner *p, const int64_t *halo_off, const int32_t *halo,
                         const int32_t *ranked) {
    p->halo_off.assign(halo_off, halo_off + p->P + 1);
    int64_t tot = p->halo_off[p->P];
    p->halo.assign(halo, halo + tot);
    p->ranked.assign(ranked, ranked + tot);
    for (int64_t i = 0; i < tot; ++i)
        if (halo[i] < 0 || halo[i] >= p->n_keys || ranked[i] < 0 || ranked[i] >= p->n_keys) {
            cg_set_error("cg_planner_set_halos: key out of range");
            return -1;
        }
    return 0;
}

// CacheSystem.warm (cache.py:323-347): local d takes the first c_gpu[d] of
// its ranked list; the global level the rank-position interleave, deduped.
int cg_planner_warm(cg_planner *p) {
    for (int d = 0; d < p->P; ++d) {
        int64_t b = p->halo_off[d], e = p->halo_off[d + 1];
        int64_t take = std::min<int64_t>(p->loc[d].capacity, e - b);
        for (int64_t i = 0; i < take; ++i) p->loc[d].insert(p->ranked[b + i], 0);
    }
    std::vector<uint8_t> seen(p->n_keys, 0);
    int64_t taken = 0, longest = 0;
    for (int d = 0; d < p->P; ++d)
        longest = std::max<int64_t>(longest, p->halo_off[d + 1] - p->halo_off[d]);
    for (int64_t pos = 0; pos < longest && taken < p->glo.capacity; ++pos)
        for (int d = 0; d < p->P && taken < p->glo.capacity; ++d) {
            int64_t b = p->halo_off[d];
            if (pos < p->halo_off[d + 1] - b) {
                int32_t k = p->ranked[b + pos];
                if (!seen[k]) { seen[k] = 1; p->glo.insert(k, 0); ++taken; }
            }
        }
    return 0;
}

int cg_planner_epoch(cg_planner *p, int epoch, int staleness, int8_t *outcome,
                     int32_t *version, int32_t *hit_slot, int32_t *slot_after,
                     int32_t *lslot_pos, uint8_t *lslot_dirty,
                     int32_t *gslot_vertex, uint8_t *gslot_dirty, int64_t *counts) {
    if (p->halo_off.empty()) { cg_set_error("cg_planner_epoch: halos not set"); return -1; }
    for (auto &L : p->loc) std::fill(L.slot_dirty.begin(), L.slot_dirty.end(), 0);
    std::fill(p->glo.slot_dirty.begin(), p->glo.slot_dirty.end(), 0);
    for (auto &L : p->loc) L.admissions = 0;
    p->glo.admissions = 0;
    std::vector<int64_t> before(3 * p->P);
    for (int d = 0; d < p->P; ++d) {
        before[3 * d] = p->lh[d];
        before[3 * d + 1] = p->gh[d];
        before[3 * d + 2] = p->ms[d];
    }
    int64_t longest = 0;
    for (int d = 0; d < p->P; ++d)
        longest = std::max<int64_t>(longest, p->halo_off[d + 1] - p->halo_off[d]);
    for (int64_t r = 0; r < longest; ++r) {
        for (int d = 0; d < p->P; ++d) {
            int64_t b = p->halo_off[d];
            if (r >= p->halo_off[d + 1] - b) continue;
            int64_t i = b + r;
            int32_t k = p->halo[i];
            int32_t served, hs;
            int o = p->lookup(d, k, epoch, staleness, &served, &hs);
            if (outcome) outcome[i] = (int8_t)o;
            if (version) version[i] = served;
            if (hit_slot) hit_slot[i] = hs;
            if (slot_after) slot_after[i] = p->loc[d].slot[k];
        }
    }
    // final slot states
    if (lslot_pos || lslot_dirty) {
        for (int d = 0; d < p->P; ++d) {
            Level &L = p->loc[d];
            // key -> position within partition d's halo (binary search: halo ascending by id,
            // and union indices are ascending with id, so keys are ascending too)
            const int32_t *hb = p->halo.data() + p->halo_off[d];
            int64_t hn = p->halo_off[d + 1] - p->halo_off[d];
            for (int64_t s = 0; s < L.capacity; ++s) {
                int64_t o = p->lslot_off[d] + s;
                int32_t k = L.slot_key[s];
                int32_t pos = -1;
                if (k >= 0 && L.slot[k] == s) {
                    const int32_t *it = std::lower_bound(hb, hb + hn, k);
                    if (it != hb + hn && *it == k) pos = (int32_t)(it - hb);
                }
                if (lslot_pos) lslot_pos[o] = pos;
                if (lslot_dirty) lslot_dirty[o] = L.slot_dirty[s];
            }
        }
    }
    if (gslot_vertex || gslot_dirty) {
        for (int64_t s = 0; s < p->glo.capacity; ++s) {
            int32_t k = p->glo.slot_key[s];
            bool live = k >= 0 && p->glo.slot[k] == s;
            if (gslot_vertex) gslot_vertex[s] = live ? k : -1;
            if (gslot_dirty) gslot_dirty[s] = p->glo.slot_dirty[s];
        }
    }
    if (counts)
        for (int d = 0; d < p->P; ++d) {
            counts[3 * d] = p->lh[d] - before[3 * d];
            counts[3 * d + 1] = p->gh[d] - before[3 * d + 1];
            counts[3 * d + 2] = p->ms[d] - before[3 * d + 2];
        }
    return 0;
}

int cg_planner_state(cg_planner *p, int32_t *req_slot, int32_t *req_ver,
                     int32_t *gslot_of_union, int32_t *glob_ver_by_slot,
                     int32_t *admissions_last_epoch, int32_t *lfree, double *lmin,
                     int32_t *gfree, double *gmin) {
    int64_t adm = p->glo.admissions;
    for (int d = 0; d < p->P; ++d) {
        Level &L = p->loc[d];
        adm += L.admissions;
        for (int64_t i = p->halo_off[d]; i < p->halo_off[d + 1]; ++i) {
            int32_t k = p->halo[i];
            if (req_slot) req_slot[i] = L.slot[k];
            if (req_ver) req_ver[i] = L.slot[k] >= 0 ? L.ver[k] : 0;
        }
        if (lfree) lfree[d] = L.admit_mode();
        if (lmin) lmin[d] = L.min_score();
    }
    if (gslot_of_union)
        for (int64_t k = 0; k < p->n_keys; ++k) gslot_of_union[k] = p->glo.slot[k];
    if (glob_ver_by_slot)
        for (int64_t s = 0; s < p->glo.capacity; ++s) {
            int32_t k = p->glo.slot_key[s];
            glob_ver_by_slot[s] = (k >= 0 && p->glo.slot[k] == s) ? p->glo.ver[k] : 0;
        }
    if (admissions_last_epoch) *admissions_last_epoch = (int32_t)adm;
    if (gfree) *gfree = p->glo.admit_mode();
    if (gmin) *gmin = p->glo.min_score();
    return 0;
}

int cg_planner_lookup(cg_planner *p, int part, int32_t vertex, int epoch, int staleness,
                      int *outcome) {
    if (part < 0 || part >= p->P) { cg_set_error("device out of range"); return -1; }
    if (vertex < 0 || vertex >= p->n_keys) { cg_set_error("vertex key out of range"); return -1; }
    int32_t served, hs;
    *outcome = p->lookup(part, vertex, epoch, staleness, &served, &hs);
    return 0;
}

int cg_planner_admit(cg_planner *p, int level, int part, int32_t vertex, int version,
                     int32_t *victim) {
    if (vertex < 0 || vertex >= p->n_keys) { cg_set_error("vertex key out of range"); return -1; }
    if (level == 0) {
        *victim = p->glo.insert(vertex, version);
        return 0;
    }
    if (part < 0 || part >= p->P) { cg_set_error("device out of range"); return -1; }
    *victim = p->loc[part].insert(vertex, version);
    return 0;
}

int cg_planner_counters(cg_planner *p, int64_t *lookups, int64_t *local_hits,
                        int64_t *global_hits, int64_t *misses) {
    for (int d = 0; d < p->P; ++d) {
        lookups[d] = p->lookups[d];
        local_hits[d] = p->lh[d];
        global_hits[d] = p->gh[d];
        misses[d] = p->ms[d];
    }
    return 0;
}

int cg_planner_occupancy(cg_planner *p, int64_t *global_count, int64_t *local_counts) {
    *global_count = p->glo.count;
    for (int d = 0; d < p->P; ++d) local_counts[d] = p->loc[d].count;
    return 0;
}

}  // extern "C"
