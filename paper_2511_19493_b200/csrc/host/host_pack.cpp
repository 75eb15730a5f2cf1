// host_pack.cpp — host side of the upload boundary (part of librfxc.so).
//
// The drop-in API receives the forest as per-tree host arrays (forest.py:67-99,
// _kernels.py:7-17) and the dataset as a column-major f64 matrix
// (dataset.py:59-71).  Instead of shipping ~25 B/node of raw arrays over PCIe
// and repacking on the device, these functions pack the traversal records
// (8 B/node f32 layout, 16 B/node f64 layout — same encoding as the device
// packer in forest.cu) and the f32 feature copy directly into caller-owned
// (pinned) host buffers with one thread per core, so only the packed bytes
// cross the bus.  Trees whose right child is not left + 1 (hand-built trees;
// trained trees always satisfy it, _kernels.py:313-317) are relaid out
// breadth-first here, keeping the reference's leaf ordinals.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/rfxc.h"

namespace rfxc {
std::string& last_error();
}

namespace {

int feature_bits(int p)
{
    int fb = 1;
    while ((1 << fb) < p) fb++;
    return fb;
}

// f64 -> f32 rounded toward -inf (exact compare for f32-representable x)
inline float round_down_f32(double t)
{
    float f = (float)t;
    if ((double)f > t) {  // step one ulp toward -inf on the bit pattern
        uint32_t u;
        std::memcpy(&u, &f, 4);
        if (f > 0.0f) u -= 1;
        else if (f < 0.0f) u += 1;
        else u = 0x80000001u;  // just below +0: the smallest negative subnormal
        std::memcpy(&f, &u, 4);
    }
    return f;
}

template <class F>
void parallel_for(int64_t count, int nthreads, F&& fn)
{
    if (nthreads <= 1 || count < 2) {
        for (int64_t i = 0; i < count; i++) fn(i);
        return;
    }
    std::vector<std::thread> ts;
    std::atomic<int64_t> next{0};
    for (int t = 0; t < nthreads; t++)
        ts.emplace_back([&] {
            for (int64_t i; (i = next.fetch_add(1)) < count;) fn(i);
        });
    for (auto& t : ts) t.join();
}

int hw_threads(int requested)
{
    if (requested > 0) return requested;
    unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}

// RFXC_NODES_F32_B2: per tree [root, pad x3], then for every internal node x
// at even depth (breadth-first over such nodes) group0(x) = [L, R, children
// pair of L (or two pads)] and, when R is internal, group1(x) = [R (a copy),
// pad, children pair of R].  Every group is 32 bytes, so the traversal fetches
// the chosen child's record and that child's children pair with one 256-bit
// load: two levels per dependent load and per L1 request.  A block root's
// record points at group0 and carries "R internal" in bit fb+1.  slots[new] =
// old node id (-1: pad); ptr/rint per old id.  Returns the record count.
int64_t b2_slots(int64_t nc, const int8_t* st, const int32_t* lf, const int32_t* rt,
                 std::vector<int64_t>& slots, std::vector<int64_t>& ptr, std::vector<uint8_t>& rint,
                 std::string& err)
{
    slots.assign({0, -1, -1, -1});
    ptr.assign(nc, 0);
    rint.assign(nc, 0);
    std::vector<uint8_t> placed(nc, 0);
    placed[0] = 1;
    int64_t nplaced = 1;
    auto internal = [&](int64_t t) { return st[t] == 0; };
    auto place = [&](int64_t o) {
        if (o <= 0 || o >= nc || placed[o]) return false;
        placed[o] = 1;
        nplaced++;
        slots.push_back(o);
        return true;
    };
    std::vector<int64_t> roots;
    if (internal(0)) roots.push_back(0);
    for (size_t q = 0; q < roots.size(); q++) {
        const int64_t x = roots[q], L = lf[x], R = rt[x];
        const int64_t g0 = (int64_t)slots.size();
        ptr[x] = g0;
        if (!place(L) || !place(R)) {
            err = "malformed children";
            return -1;
        }
        rint[x] = internal(R) ? 1 : 0;
        if (internal(L)) {
            ptr[L] = g0 + 2;
            if (!place(lf[L]) || !place(rt[L])) {
                err = "malformed children";
                return -1;
            }
            for (int64_t g : {(int64_t)lf[L], (int64_t)rt[L]})
                if (internal(g)) roots.push_back(g);
        } else {
            slots.push_back(-1);
            slots.push_back(-1);
        }
        if (internal(R)) {
            ptr[R] = (int64_t)slots.size() + 2;
            slots.push_back(R);  // the copy; R's own slot is group0's second
            slots.push_back(-1);
            if (!place(lf[R]) || !place(rt[R])) {
                err = "malformed children";
                return -1;
            }
            for (int64_t g : {(int64_t)lf[R], (int64_t)rt[R]})
                if (internal(g)) roots.push_back(g);
        }
    }
    if (nplaced != nc) {
        err = "unreachable nodes";
        return -1;
    }
    return (int64_t)slots.size();
}

int pack_b2(const void* const* status, const void* const* split_var, const void* const* threshold,
            const void* const* cat_mask, const void* const* left, const void* const* right,
            const int64_t* node_counts, int32_t B, const uint8_t* col_cat, int32_t p, void* h_nodes,
            int64_t* h_node_off, int32_t* h_leaf_counts, int32_t nthreads)
{
    const int fb = feature_bits(p);
    const int64_t max_ptr = int64_t(1) << (30 - fb);
    std::vector<std::string> errs(B);
    std::vector<int64_t> cnt(B, 0);
    const int T = hw_threads(nthreads);
    // pass 1: record counts (h_nodes == nullptr: sizing call, stop here)
    parallel_for(B, T, [&](int64_t b) {
        std::vector<int64_t> slots, ptr;
        std::vector<uint8_t> rint;
        std::string err;
        cnt[b] = b2_slots(node_counts[b], static_cast<const int8_t*>(status[b]),
                          static_cast<const int32_t*>(left[b]), static_cast<const int32_t*>(right[b]), slots,
                          ptr, rint, err);
        if (cnt[b] < 0) errs[b] = "tree " + std::to_string(b) + ": " + err;
        int32_t nleaf = 0;
        const int8_t* st = static_cast<const int8_t*>(status[b]);
        for (int64_t t = 0; t < node_counts[b]; t++) nleaf += st[t] == 1;
        h_leaf_counts[b] = nleaf;
    });
    for (int b = 0; b < B; b++)
        if (!errs[b].empty()) {
            rfxc::last_error() = errs[b];
            return RFXC_EDATA;
        }
    h_node_off[0] = 0;
    for (int b = 0; b < B; b++) h_node_off[b + 1] = h_node_off[b] + cnt[b];
    if (!h_nodes) return RFXC_OK;
    parallel_for(B, T, [&](int64_t b) {
        const int64_t nc = node_counts[b];
        const int8_t* st = static_cast<const int8_t*>(status[b]);
        const int32_t* sv = static_cast<const int32_t*>(split_var[b]);
        const double* th = static_cast<const double*>(threshold[b]);
        const int64_t* cm = static_cast<const int64_t*>(cat_mask[b]);
        const int32_t* lf = static_cast<const int32_t*>(left[b]);
        const int32_t* rt = static_cast<const int32_t*>(right[b]);
        std::vector<int64_t> slots, ptr;
        std::vector<uint8_t> rint;
        std::string err;
        b2_slots(nc, st, lf, rt, slots, ptr, rint, err);
        std::vector<int32_t> code(nc, -1);
        int32_t nleaf = 0;
        for (int64_t t = 0; t < nc; t++)
            if (st[t] == 1) code[t] = nleaf++;
        uint32_t* out = static_cast<uint32_t*>(h_nodes) + 2 * h_node_off[b];
        for (size_t t = 0; t < slots.size(); t++) {
            const int64_t o = slots[t];
            uint32_t x = 0u, y = 0u;
            if (o >= 0 && st[o] == 1) {
                x = (uint32_t)code[o];
            } else if (o >= 0) {
                const int f = sv[o];
                if (f < 0 || f >= p) {
                    errs[b] = "tree " + std::to_string(b) + ": split_var out of range";
                    return;
                }
                if (ptr[o] >= max_ptr) {
                    errs[b] = "tree " + std::to_string(b) + ": child id out of range for layout";
                    return;
                }
                const bool cat = col_cat[f] == 1;
                if (cat) {
                    x = (uint32_t)(cm[o] & 0xffffffffLL);
                } else {
                    const float fr = round_down_f32(th[o]);
                    std::memcpy(&x, &fr, 4);
                }
                y = ((uint32_t)ptr[o] << (fb + 2)) | ((uint32_t)rint[o] << (fb + 1)) | ((uint32_t)cat << fb) |
                    (uint32_t)f;
            }
            out[2 * t] = x;
            out[2 * t + 1] = y;
        }
    });
    for (int b = 0; b < B; b++)
        if (!errs[b].empty()) {
            rfxc::last_error() = errs[b];
            return RFXC_EDATA;
        }
    return RFXC_OK;
}

}  // namespace

extern "C" int rfxc_forest_pack_host(const void* const* status, const void* const* split_var,
                                     const void* const* threshold, const void* const* cat_mask,
                                     const void* const* left, const void* const* right,
                                     const int64_t* node_counts, int32_t B,
                                     const uint8_t* col_cat, int32_t p, int32_t layout,
                                     void* h_nodes, int64_t* h_node_off,
                                     int32_t* h_leaf_counts, int32_t nthreads)
{
    if (B < 1 || p < 1) {
        rfxc::last_error() = "forest_pack_host: bad shape";
        return RFXC_EDATA;
    }
    if (layout != RFXC_NODES_F32 && layout != RFXC_NODES_F64 && layout != RFXC_NODES_F32_B2) {
        rfxc::last_error() = "forest_pack_host: unknown layout " + std::to_string(layout);
        return RFXC_EDATA;
    }
    if (layout == RFXC_NODES_F32_B2)
        return pack_b2(status, split_var, threshold, cat_mask, left, right, node_counts, B, col_cat, p,
                       h_nodes, h_node_off, h_leaf_counts, nthreads);
    h_node_off[0] = 0;
    for (int b = 0; b < B; b++) h_node_off[b + 1] = h_node_off[b] + node_counts[b];
    const int fb = feature_bits(p);
    const int64_t max_left = layout == RFXC_NODES_F32 ? (int64_t(1) << (31 - fb)) : INT32_MAX;
    std::vector<std::string> errs(B);
    parallel_for(B, hw_threads(nthreads), [&](int64_t b) {
        const int64_t nc = node_counts[b];
        const int8_t* st = static_cast<const int8_t*>(status[b]);
        const int32_t* sv = static_cast<const int32_t*>(split_var[b]);
        const double* th = static_cast<const double*>(threshold[b]);
        const int64_t* cm = static_cast<const int64_t*>(cat_mask[b]);
        const int32_t* lf = static_cast<const int32_t*>(left[b]);
        const int32_t* rt = static_cast<const int32_t*>(right[b]);
        // order[new] = old node id; identity when siblings are adjacent
        std::vector<int64_t> order;
        bool adjacent = true;
        for (int64_t t = 0; t < nc && adjacent; t++)
            if (st[t] == 0 && rt[t] != lf[t] + 1) adjacent = false;
        std::vector<int32_t> code(nc, -1);
        int32_t nleaf = 0;
        for (int64_t t = 0; t < nc; t++)
            if (st[t] == 1) code[t] = nleaf++;
        h_leaf_counts[b] = nleaf;
        std::vector<int64_t> newid;
        if (!adjacent) {
            order.reserve(nc);
            newid.assign(nc, -1);
            order.push_back(0);
            newid[0] = 0;
            for (size_t q = 0; q < order.size(); q++) {
                const int64_t o = order[q];
                if (st[o] == 0) {
                    for (int64_t ch : {(int64_t)lf[o], (int64_t)rt[o]}) {
                        if (ch <= 0 || ch >= nc || newid[ch] >= 0) {
                            errs[b] = "tree " + std::to_string(b) + ": malformed children";
                            return;
                        }
                        newid[ch] = (int64_t)order.size();
                        order.push_back(ch);
                    }
                }
            }
            if ((int64_t)order.size() != nc) {
                errs[b] = "tree " + std::to_string(b) + ": unreachable nodes";
                return;
            }
        }
        const int64_t base = h_node_off[b];
        for (int64_t t = 0; t < nc; t++) {
            const int64_t o = adjacent ? t : order[t];
            const bool leaf = st[o] == 1;
            const int64_t l = leaf ? 0 : (adjacent ? lf[o] : newid[lf[o]]);
            if (!leaf && (l < 1 || l >= max_left)) {
                errs[b] = "tree " + std::to_string(b) + ": child id out of range for layout";
                return;
            }
            const int f = leaf ? 0 : sv[o];
            if (!leaf && (f < 0 || f >= p)) {
                errs[b] = "tree " + std::to_string(b) + ": split_var out of range";
                return;
            }
            const bool cat = !leaf && col_cat[f] == 1;
            if (layout == RFXC_NODES_F32) {
                uint32_t x, y;
                if (leaf) {
                    x = (uint32_t)code[o];
                    y = 0u;
                } else {
                    if (cat) {
                        x = (uint32_t)(cm[o] & 0xffffffffLL);
                    } else {
                        float fr = round_down_f32(th[o]);
                        std::memcpy(&x, &fr, 4);
                    }
                    y = ((uint32_t)l << (fb + 1)) | ((uint32_t)cat << fb) | (uint32_t)f;
                }
                uint32_t* rec = static_cast<uint32_t*>(h_nodes) + 2 * (base + t);
                rec[0] = x;
                rec[1] = y;
            } else {
                int32_t* rec = static_cast<int32_t*>(h_nodes) + 4 * (base + t);
                if (leaf) {
                    rec[0] = rec[1] = 0;
                    rec[2] = -1;
                    rec[3] = code[o];
                } else {
                    int64_t bits;
                    if (cat) bits = cm[o];
                    else std::memcpy(&bits, &th[o], 8);
                    rec[0] = (int32_t)(bits & 0xffffffffLL);
                    rec[1] = (int32_t)(bits >> 32);
                    rec[2] = f | ((int)cat << 30);
                    rec[3] = (int32_t)l;
                }
            }
        }
    });
    for (int b = 0; b < B; b++)
        if (!errs[b].empty()) {
            rfxc::last_error() = errs[b];
            return RFXC_EDATA;
        }
    return RFXC_OK;
}

extern "C" int rfxc_values_to_f32_host(const double* h_values, int64_t count, float* h_out,
                                       int32_t* exact, int32_t nthreads)
{
    const int T = hw_threads(nthreads);
    const int64_t chunk = (count + T - 1) / T;
    std::vector<int> bad(T, 0);
    parallel_for(T, T, [&](int64_t t) {
        const int64_t lo = t * chunk, hi = std::min(count, lo + chunk);
        int b = 0;
        for (int64_t i = lo; i < hi; i++) {
            const float f = (float)h_values[i];
            h_out[i] = f;
            b |= ((double)f != h_values[i]);
        }
        bad[t] = b;
    });
    int any = 0;
    for (int b : bad) any |= b;
    *exact = !any;
    return RFXC_OK;
}
