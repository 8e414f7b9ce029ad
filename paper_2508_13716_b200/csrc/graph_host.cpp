// Native integer preprocessing for the hot path's inputs:
// CSR construction, k-hop halos, partition statistics and the fp64 influence
// scores.  Results are bit-identical to halopart's numpy code
// (graph.py:24-129, 203-228, 298-335; partitioner.py:324-345): integer work
// is exact, and the influence sums are sequential in CSR order, which is the
// order np.bincount accumulates in, with plain IEEE mul/sqrt/div (this file
// is compiled without FMA contraction).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/capgnn.h"

extern void cg_set_error(const std::string &msg);

extern "C" {

// Deduplicate (src, dst) pairs and emit both CSR directions, rows ascending.
// out_off/in_off: [n+1]; out_tgt/in_tgt: capacity m; *n_edges = unique count.
int cg_csr_from_pairs(int64_t n, int64_t m, const int64_t *src, const int64_t *dst,
                      int64_t *out_off, int64_t *out_tgt, int64_t *in_off, int64_t *in_tgt,
                      int64_t *n_edges) {
    std::vector<int64_t> code(m);
    for (int64_t i = 0; i < m; ++i) {
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) {
            cg_set_error("edge endpoint outside 0..n_vertices-1");
            return -1;
        }
        code[i] = src[i] * n + dst[i];
    }
    std::sort(code.begin(), code.end());
    code.erase(std::unique(code.begin(), code.end()), code.end());
    const int64_t E = (int64_t)code.size();
    std::fill(out_off, out_off + n + 1, 0);
    std::fill(in_off, in_off + n + 1, 0);
    for (int64_t i = 0; i < E; ++i) {
        ++out_off[code[i] / n + 1];
        ++in_off[code[i] % n + 1];
    }
    for (int64_t v = 0; v < n; ++v) {
        out_off[v + 1] += out_off[v];
        in_off[v + 1] += in_off[v];
    }
    std::vector<int64_t> fill(in_off, in_off + n);
    for (int64_t i = 0; i < E; ++i) {  // codes ascending: (src, dst) order
        int64_t s = code[i] / n, d = code[i] % n;
        out_tgt[i] = d;
        in_tgt[fill[d]++] = s;  // within a dst row, src ascending
    }
    *n_edges = E;
    return 0;
}

// Undirected neighbour lists (union of out and in lists, deduplicated).
// und_off: [n+1]; und_tgt capacity out_off[n] + in_off[n].
int cg_undirected_csr(int64_t n, const int64_t *out_off, const int64_t *out_tgt,
                      const int64_t *in_off, const int64_t *in_tgt, int64_t *und_off,
                      int64_t *und_tgt) {
    und_off[0] = 0;
    int64_t w = 0;
    for (int64_t v = 0; v < n; ++v) {
        const int64_t *a = out_tgt + out_off[v], *ae = out_tgt + out_off[v + 1];
        const int64_t *b = in_tgt + in_off[v], *be = in_tgt + in_off[v + 1];
        while (a < ae || b < be) {  // merge two ascending lists without duplicates
            int64_t x;
            if (b >= be || (a < ae && *a < *b)) x = *a++;
            else if (a >= ae || *b < *a) x = *b++;
            else { x = *a++; ++b; }
            und_tgt[w++] = x;
        }
        und_off[v + 1] = w;
    }
    return 0;
}

// Halo of one partition: vertices outside it within `hops` undirected steps,
// written ascending into out (capacity n); *n_out = count.
int cg_khop_halo(int64_t n, const int64_t *und_off, const int64_t *und_tgt,
                 const int32_t *parts, int32_t part, int hops, int32_t *out, int64_t *n_out) {
    if (hops < 1) { cg_set_error("hops must be >= 1"); return -1; }
    std::vector<uint8_t> seen(n, 0);
    std::vector<int64_t> frontier, next;
    for (int64_t v = 0; v < n; ++v)
        if (parts[v] == part) { seen[v] = 2; frontier.push_back(v); }
    if (frontier.empty()) { cg_set_error("inner set is empty"); return -1; }
    for (int h = 0; h < hops && !frontier.empty(); ++h) {
        next.clear();
        for (int64_t v : frontier)
            for (int64_t e = und_off[v]; e < und_off[v + 1]; ++e) {
                int64_t u = und_tgt[e];
                if (!seen[u]) { seen[u] = 1; next.push_back(u); }
            }
        frontier.swap(next);
    }
    int64_t c = 0;
    for (int64_t v = 0; v < n; ++v)
        if (seen[v] == 1) out[c++] = (int32_t)v;
    *n_out = c;
    return 0;
}

// cut_edges[i]: directed edges with exactly one endpoint in partition i;
// all_edges[i]: edges with both endpoints in inner_i | halo_i.
int cg_partition_stats(int64_t n, const int64_t *out_off, const int64_t *out_tgt,
                       const int32_t *parts, int P, const int64_t *halo_off,
                       const int32_t *halo, int64_t *cut, int64_t *all_edges) {
    std::vector<int64_t> c(P, 0);
    for (int64_t u = 0; u < n; ++u)
        for (int64_t e = out_off[u]; e < out_off[u + 1]; ++e) {
            int32_t pa = parts[u], pb = parts[out_tgt[e]];
            if (pa != pb) { ++c[pa]; ++c[pb]; }
        }
    std::vector<uint8_t> mem(n);
    for (int i = 0; i < P; ++i) {
        cut[i] = c[i];
        for (int64_t v = 0; v < n; ++v) mem[v] = parts[v] == i;
        for (int64_t k = halo_off[i]; k < halo_off[i + 1]; ++k) mem[halo[k]] = 1;
        int64_t a = 0;
        for (int64_t u = 0; u < n; ++u)
            if (mem[u])
                for (int64_t e = out_off[u]; e < out_off[u + 1]; ++e) a += mem[out_tgt[e]];
        all_edges[i] = a;
    }
    return 0;
}

// Per-vertex influence terms over ALL vertices (caller multiplies by overlap):
// out_term[u] = sum_{u->v} 1/sqrt(dout(u) din(v)), in ascending v;
// in_term[v]  = sum_{u->v} 1/sqrt(dout(u) din(v)), in ascending u.
int cg_influence_terms(int64_t n, const int64_t *out_off, const int64_t *out_tgt,
                       const int64_t *in_off, const int64_t *in_tgt, double *out_term,
                       double *in_term) {
    for (int64_t u = 0; u < n; ++u) {
        double du = (double)(out_off[u + 1] - out_off[u]);
        double s = 0.0;
        for (int64_t e = out_off[u]; e < out_off[u + 1]; ++e) {
            int64_t v = out_tgt[e];
            double den = du * (double)(in_off[v + 1] - in_off[v]);
            s += den > 0 ? 1.0 / std::sqrt(den) : 0.0;
        }
        out_term[u] = s;
    }
    for (int64_t v = 0; v < n; ++v) {
        double dv = (double)(in_off[v + 1] - in_off[v]);
        double s = 0.0;
        for (int64_t e = in_off[v]; e < in_off[v + 1]; ++e) {
            int64_t u = in_tgt[e];
            double den = (double)(out_off[u + 1] - out_off[u]) * dv;
            s += den > 0 ? 1.0 / std::sqrt(den) : 0.0;
        }
        in_term[v] = s;
    }
    return 0;
}

}  // extern "C"
