// rfx_train.cpp — input producer: the reference CPU trainer restated in C++.
//
// The proximity hot path takes "the forest grown by the reference's CPU
// trainer with the same seed" as its input (BASELINE.json north_star).  The
// reference trainer is Python + Numba and does not exist on the GPU box, so
// this file restates it (bit-exact forest bytes, checked against the
// reference's RFX1 output in tests/test_train.py) to regenerate the input
// forest there.  It is NOT on the hot path and never timed by bench.py.
//
//   bootstrap            _kernels.py:28-34  (n bounded draws, SEQ_TREE stream)
//   node statistics      _kernels.py:200-232
//   feature subset       _kernels.py:236-238, rng.py:90-99 (partial shuffle)
//   numeric split scan   _kernels.py:46-105  (ties on delta keep smallest tau)
//   categorical scan     _kernels.py:108-159 (canonical masks, bit 0 set)
//   split selection      _kernels.py:240-274 (ties keep the lower feature)
//   stable partition     _kernels.py:284-311; children appended (lc, lc+1)
//   OOB votes            _kernels.py:377-385, forest.py:287-290
//
// All floating-point expressions keep the reference's operation order and
// are compiled with -ffp-contract=off so results match LLVM/Numba bitwise.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "pcg32.h"

namespace {

struct TreeOut {
    std::vector<int8_t> status;
    std::vector<int32_t> split_var, left, right, node_class, node_raw;
    std::vector<double> threshold;
    std::vector<int64_t> cat_mask, class_pops, node_weight;
    std::vector<int32_t> inbag;
    int error = 0;
};

struct Problem {
    const double* values;   // (n, p) column-major
    const int32_t* labels;
    const uint8_t* col_cat;
    const int32_t* col_levels;
    int64_t n;
    int32_t p, C, mtry, min_node_size;
    int64_t max_nodes;
};

struct Triple {
    double v;
    int32_t y;
    int32_t w;
};

inline double gini_of(const int64_t* counts, int64_t total, int C)
{
    double s = 0.0;
    for (int c = 0; c < C; c++) {
        double f = (double)counts[c] / (double)total;
        s += f * f;
    }
    return 1.0 - s;
}

// _kernels.py:46-105
void threshold_scan(int64_t m, Triple* buf, const int64_t* pops,
                    int64_t* left_counts, int C, double ip, int64_t wtot,
                    double* out_delta, double* out_tau)
{
    // any sort order among equal values gives the same scan: the criterion
    // is only evaluated between distinct values and the counts are integers.
    std::sort(buf, buf + m, [](const Triple& a, const Triple& b) { return a.v < b.v; });
    for (int c = 0; c < C; c++) left_counts[c] = 0;
    int64_t lw = 0;
    double best_delta = -1.0, best_tau = 0.0;
    for (int64_t k = 0; k + 1 < m; k++) {
        left_counts[buf[k].y] += buf[k].w;
        lw += buf[k].w;
        if (buf[k].v < buf[k + 1].v) {
            int64_t rw = wtot - lw;
            double il = 0.0, ir = 0.0;
            for (int c = 0; c < C; c++) {
                double fl = (double)left_counts[c] / (double)lw;
                double fr = (double)(pops[c] - left_counts[c]) / (double)rw;
                il += fl * fl;
                ir += fr * fr;
            }
            il = 1.0 - il;
            ir = 1.0 - ir;
            double delta = ip - ((double)lw / (double)wtot) * il
                              - ((double)rw / (double)wtot) * ir;
            if (delta > best_delta) {
                best_delta = delta;
                best_tau = buf[k].v;
            }
        }
    }
    *out_delta = best_delta;
    *out_tau = best_tau;
}

// _kernels.py:108-159
void garside_scan(int64_t m, const Triple* buf, int n_levels, int64_t* lvl_counts,
                  int64_t* lvl_w, int64_t* left_counts, const int64_t* pops, int C,
                  double ip, int64_t wtot, double* out_delta, int64_t* out_mask)
{
    for (int k = 0; k < n_levels; k++) {
        lvl_w[k] = 0;
        for (int c = 0; c < C; c++) lvl_counts[k * C + c] = 0;
    }
    for (int64_t t = 0; t < m; t++) {
        int code = (int)buf[t].v;
        lvl_counts[code * C + buf[t].y] += buf[t].w;
        lvl_w[code] += buf[t].w;
    }
    int present = 0;
    for (int k = 0; k < n_levels; k++) present += lvl_w[k] > 0;
    if (present < 2) {
        *out_delta = -1.0;
        *out_mask = 0;
        return;
    }
    int64_t full = ((int64_t)1 << n_levels) - 1;
    double best_delta = -1.0;
    int64_t best_mask = 0;
    for (int64_t mask = 1; mask < full; mask += 2) {
        int64_t lw = 0;
        for (int c = 0; c < C; c++) left_counts[c] = 0;
        for (int k = 0; k < n_levels; k++) {
            if ((mask >> k) & 1) {
                lw += lvl_w[k];
                for (int c = 0; c < C; c++) left_counts[c] += lvl_counts[k * C + c];
            }
        }
        int64_t rw = wtot - lw;
        if (lw > 0 && rw > 0) {
            double il = 0.0, ir = 0.0;
            for (int c = 0; c < C; c++) {
                double fl = (double)left_counts[c] / (double)lw;
                double fr = (double)(pops[c] - left_counts[c]) / (double)rw;
                il += fl * fl;
                ir += fr * fr;
            }
            double delta = ip - ((double)lw / (double)wtot) * (1.0 - il)
                              - ((double)rw / (double)wtot) * (1.0 - ir);
            if (delta > best_delta) {
                best_delta = delta;
                best_mask = mask;
            }
        }
    }
    *out_delta = best_delta;
    *out_mask = best_mask;
}

inline bool goes_left(bool is_cat, double v, int64_t mask, double tau)
{
    return is_cat ? (((mask >> (int64_t)v) & 1) == 1) : (v <= tau);
}

// _kernels.py:162-330
void grow(const Problem& P, int64_t tree_seed, TreeOut& T)
{
    const int64_t n = P.n;
    const int C = P.C;
    const int64_t mn = P.max_nodes;
    std::vector<int32_t> idx;
    for (int64_t i = 0; i < n; i++)
        if (T.inbag[i] > 0) idx.push_back((int32_t)i);
    const int64_t total = (int64_t)idx.size();

    std::vector<int32_t> node_start(1, 0), node_end(1, (int32_t)total);
    std::vector<int64_t> feat(P.p);
    std::vector<Triple> buf(std::max<int64_t>(total, 1));
    std::vector<int32_t> tmp(std::max<int64_t>(total, 1));
    std::vector<int64_t> pops(C), left_counts(C), lvl_counts(32 * C), lvl_w(32);

    uint64_t st[2];
    rfx_pcg32_make(tree_seed, RFX_SEQ_GROW, st);

    int64_t count = 1;
    auto push_leaf_fields = [&](int64_t m, int64_t w, int best_c) {
        T.node_class.push_back(best_c);
        T.node_raw.push_back((int32_t)m);
        T.node_weight.push_back(w);
        for (int c = 0; c < C; c++) T.class_pops.push_back(pops[c]);
    };
    for (int64_t node = 0; node < count; node++) {
        int32_t start = node_start[node], end = node_end[node];
        int64_t m = end - start;
        for (int c = 0; c < C; c++) pops[c] = 0;
        int64_t w = 0;
        for (int32_t t = start; t < end; t++) {
            int32_t i = idx[t];
            pops[P.labels[i]] += T.inbag[i];
            w += T.inbag[i];
        }
        int best_c = 0;
        for (int c = 1; c < C; c++)
            if (pops[c] > pops[best_c]) best_c = c;
        push_leaf_fields(m, w, best_c);

        auto make_terminal = [&]() {
            T.status.push_back(1);
            T.split_var.push_back(-1);
            T.threshold.push_back(0.0);
            T.cat_mask.push_back(0);
            T.left.push_back(-1);
            T.right.push_back(-1);
        };
        bool pure = pops[best_c] == w;
        if (pure || w < P.min_node_size || m < 2) {
            make_terminal();
            continue;
        }
        double ip = gini_of(pops.data(), w, C);
        for (int j = 0; j < P.p; j++) feat[j] = j;
        for (int t = 0; t < P.mtry; t++) {   // rng.py:90-99
            int64_t j = t + (int64_t)rfx_pcg32_bounded(st, (uint32_t)(P.p - t));
            std::swap(feat[t], feat[j]);
        }
        bool found = false;
        double best_delta = 0.0, best_tau = 0.0;
        int best_feat = -1;
        int64_t best_mask = 0;
        for (int f = 0; f < P.mtry; f++) {
            int j = (int)feat[f];
            const double* col = P.values + (int64_t)j * n;
            for (int32_t t = start; t < end; t++) {
                int32_t i = idx[t];
                buf[t - start] = Triple{col[i], P.labels[i], T.inbag[i]};
            }
            double delta, tau = 0.0;
            int64_t mask = 0;
            if (P.col_cat[j] == 1)
                garside_scan(m, buf.data(), P.col_levels[j], lvl_counts.data(),
                             lvl_w.data(), left_counts.data(), pops.data(), C, ip,
                             w, &delta, &mask);
            else
                threshold_scan(m, buf.data(), pops.data(), left_counts.data(), C,
                               ip, w, &delta, &tau);
            if (delta > 0.0) {
                bool better = !found || delta > best_delta ||
                              (delta == best_delta && j < best_feat);
                if (better) {
                    found = true;
                    best_delta = delta;
                    best_feat = j;
                    best_tau = tau;
                    best_mask = mask;
                }
            }
        }
        if (!found) {
            make_terminal();
            continue;
        }
        bool is_cat = P.col_cat[best_feat] == 1;
        const double* col = P.values + (int64_t)best_feat * n;
        int32_t nl = 0;
        for (int32_t t = start; t < end; t++)
            nl += goes_left(is_cat, col[idx[t]], best_mask, best_tau);
        int32_t a = 0, b = nl;
        for (int32_t t = start; t < end; t++) {
            int32_t i = idx[t];
            if (goes_left(is_cat, col[i], best_mask, best_tau)) tmp[a++] = i;
            else tmp[b++] = i;
        }
        std::memcpy(idx.data() + start, tmp.data(), sizeof(int32_t) * m);
        if (count + 2 > mn) {
            T.error = 1;
            return;
        }
        int64_t lc = count;
        count += 2;
        node_start.push_back(start);
        node_end.push_back(start + nl);
        node_start.push_back(start + nl);
        node_end.push_back(end);
        T.status.push_back(0);
        T.split_var.push_back(best_feat);
        T.threshold.push_back(best_tau);
        T.cat_mask.push_back(best_mask);
        T.left.push_back((int32_t)lc);
        T.right.push_back((int32_t)(lc + 1));
    }
}

int32_t descend(const TreeOut& T, const Problem& P, int64_t i)
{
    int32_t node = 0;
    while (T.status[node] == 0) {
        int j = T.split_var[node];
        double v = P.values[(int64_t)j * P.n + i];
        bool go = goes_left(P.col_cat[j] == 1, v, T.cat_mask[node], T.threshold[node]);
        node = go ? T.left[node] : T.right[node];
    }
    return node;
}

struct Forest {
    std::vector<TreeOut> trees;
    std::vector<int64_t> oob_votes;
    std::string error;
};

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* rfxt_last_error(void) { return g_err.c_str(); }

// Grow trees [first_tree, first_tree + ntree) of a forest (forest.py:262-302;
// tree t uses streams seeded iseed + t, so any tree range of the forest can
// be grown independently — each GPU rank grows only its shard).  Returns an
// opaque handle or NULL (rfxt_last_error() says why).  nthreads <= 0 uses
// every core.  OOB votes cover the grown trees only.
void* rfxt_train(const double* values, int64_t n, int32_t p, const int32_t* labels,
                 int32_t n_classes, const uint8_t* col_cat, const int32_t* col_levels,
                 int32_t first_tree, int32_t ntree, int32_t mtry, int64_t iseed,
                 int32_t min_node_size, int64_t max_nodes, int32_t nthreads)
{
    Problem P{values, labels, col_cat, col_levels, n, p, n_classes, mtry,
              min_node_size, max_nodes};
    auto* F = new Forest();
    F->trees.resize(ntree);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int32_t t = 0; t < ntree; t++) {
        TreeOut& T = F->trees[t];
        T.inbag.assign(n, 0);
        uint64_t st[2];
        const int64_t tree_seed = iseed + first_tree + t;
        rfx_pcg32_make(tree_seed, RFX_SEQ_TREE, st);
        for (int64_t d = 0; d < n; d++) T.inbag[rfx_pcg32_bounded(st, (uint32_t)n)] += 1;
        grow(P, tree_seed, T);
    }
    for (int32_t t = 0; t < ntree; t++) {
        if (F->trees[t].error) {
            g_err = "tree " + std::to_string(first_tree + t) + ": exceeded max_nodes=" +
                    std::to_string(max_nodes);
            delete F;
            return nullptr;
        }
    }
    F->oob_votes.assign(n * n_classes, 0);
    for (int32_t t = 0; t < ntree; t++) {
        const TreeOut& T = F->trees[t];
        for (int64_t i = 0; i < n; i++)
            if (T.inbag[i] == 0) F->oob_votes[i * n_classes + T.node_class[descend(T, P, i)]] += 1;
    }
    return F;
}

void rfxt_node_counts(void* h, int64_t* out)
{
    auto* F = static_cast<Forest*>(h);
    for (size_t t = 0; t < F->trees.size(); t++) out[t] = (int64_t)F->trees[t].status.size();
}

// Copy the concatenated node arrays (tree-major), bootstrap counts (B, n)
// and OOB votes (n, C) into caller buffers.
void rfxt_copy(void* h, int8_t* status, int32_t* split_var, double* threshold,
               int64_t* cat_mask, int32_t* left, int32_t* right, int32_t* node_class,
               int64_t* class_pops, int32_t* node_raw, int64_t* node_weight,
               int32_t* inbag, int64_t* oob_votes)
{
    auto* F = static_cast<Forest*>(h);
    int64_t o = 0, oc = 0, ob = 0;
    for (const TreeOut& T : F->trees) {
        size_t m = T.status.size();
        std::memcpy(status + o, T.status.data(), m);
        std::memcpy(split_var + o, T.split_var.data(), 4 * m);
        std::memcpy(threshold + o, T.threshold.data(), 8 * m);
        std::memcpy(cat_mask + o, T.cat_mask.data(), 8 * m);
        std::memcpy(left + o, T.left.data(), 4 * m);
        std::memcpy(right + o, T.right.data(), 4 * m);
        std::memcpy(node_class + o, T.node_class.data(), 4 * m);
        std::memcpy(node_raw + o, T.node_raw.data(), 4 * m);
        std::memcpy(node_weight + o, T.node_weight.data(), 8 * m);
        std::memcpy(class_pops + oc, T.class_pops.data(), 8 * T.class_pops.size());
        std::memcpy(inbag + ob, T.inbag.data(), 4 * T.inbag.size());
        o += (int64_t)m;
        oc += (int64_t)T.class_pops.size();
        ob += (int64_t)T.inbag.size();
    }
    std::memcpy(oob_votes, F->oob_votes.data(), 8 * F->oob_votes.size());
}

void rfxt_free(void* h) { delete static_cast<Forest*>(h); }

}  // extern "C"
