// Memory-lean execution of the hybrid recompression (SURVEY §7.4 rules 2-7): the
// shard's row pairs are processed in chunks of whole subtrees below the top active level, so that
// only the data that crosses chunks persists on the device:
//   persistent  basis weights R_tc of the DIRECT row basis pairs (those a block references, as
//               (t,c) or, through the adjoint symmetry NEXT-1, as (s,-c)); for a leaf with #t <= k
//               that is V_tc itself (R = V, P = I, Eq. 18); the Kronecker transfer factors; and the
//               outputs as they are produced: Q/F compacted to the adaptive ranks, C_tc of the direct
//               pairs (projection), S~_b (allocated once all ranks are known);
//   per chunk   leaf V (regenerated), R of non-direct pairs, Zhat (total weights -> truncation),
//               S_b (regenerated for block weights / total weights, and again for the projection),
//               C/Q of one level in bound layout before compaction.
// Every per-pair computation is the one of the full plan, with the same kernels and inputs, so the
// results are bitwise those of the full plan (tests/test_gpu_lean.py).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

#include "dh2_shard.h"

namespace dh2 {

// ------------------------------------------------------------------ CUDA VMM (driver entry points)
namespace {
struct VmmApi {
    bool ok = false;
    CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
};

VmmApi& vmm() {
    static VmmApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    auto get = [](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q;
        return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
    };
    api.ok = get("cuMemGetAllocationGranularity", (void**)&api.MemGetAllocationGranularity) &&
             get("cuMemAddressReserve", (void**)&api.MemAddressReserve) && get("cuMemAddressFree", (void**)&api.MemAddressFree) &&
             get("cuMemCreate", (void**)&api.MemCreate) && get("cuMemRelease", (void**)&api.MemRelease) &&
             get("cuMemMap", (void**)&api.MemMap) && get("cuMemUnmap", (void**)&api.MemUnmap) &&
             get("cuMemSetAccess", (void**)&api.MemSetAccess);
    return api;
}

CUmemAllocationProp vmm_prop(int dev) {
    CUmemAllocationProp prop;
    std::memset(&prop, 0, sizeof(prop));
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    return prop;
}

#define VK(x)                                                                                            \
    do {                                                                                                 \
        CUresult r_ = (x);                                                                               \
        if (r_ == CUDA_ERROR_OUT_OF_MEMORY) throw NoMem(std::string(#x) + ": out of device memory");       \
        if (r_ != CUDA_SUCCESS) throw CudaError(std::string(#x) + " failed (CUresult " + std::to_string((int)r_) + ")"); \
    } while (0)
}  // namespace

void VaPool::reserve(int device, int nregions, size_t rbytes) {
    release();
    VmmApi& a = vmm();
    if (!a.ok) throw CudaError("CUDA virtual memory management entry points unavailable");
    dev = device;
    CUmemAllocationProp prop = vmm_prop(dev);
    VK(a.MemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    region_bytes = (rbytes + gran - 1) / gran * gran;
    CUdeviceptr p = 0;
    VK(a.MemAddressReserve(&p, region_bytes * nregions, 0, 0, 0));
    base = p;
    mapped_end.assign(nregions, 0);
}

void VaPool::ensure(int region, size_t bytes) {
    if (bytes <= mapped_end[region]) return;
    VmmApi& a = vmm();
    if (bytes > region_bytes) throw NoMem("lean plan: a device pool region exceeds its reservation");
    // grow in steps of >= 1/16 of the request (fewer mappings), rounded to the granularity
    size_t want = std::max(bytes - mapped_end[region], std::min(region_bytes - mapped_end[region], (size_t)256 << 20));
    want = (want + gran - 1) / gran * gran;
    want = std::min(want, region_bytes - mapped_end[region]);
    CUmemAllocationProp prop = vmm_prop(dev);
    CUmemGenericAllocationHandle h;
    CUresult r = a.MemCreate(&h, want, &prop, 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY) {
        // memory held in reserve by the stream-ordered pool of earlier contexts: give it back and retry
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            cudaDeviceSynchronize();
            cudaMemPoolTrimTo(pool, 0);
        }
        r = a.MemCreate(&h, want, &prop, 0);
    }
    VK(r);
    const size_t off = region * region_bytes + mapped_end[region];
    VK(a.MemMap(base + off, want, 0, h, 0));
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    VK(a.MemSetAccess(base + off, want, &acc, 1));
    maps.push_back({off, want, (unsigned long long)h});
    mapped_end[region] += want;
}

size_t VaPool::mapped_bytes() const {
    size_t b = 0;
    for (auto& m : maps) b += m.len;
    return b;
}

void VaPool::release() {
    if (!base) return;
    VmmApi& a = vmm();
    cudaDeviceSynchronize();
    for (auto& m : maps) {
        a.MemUnmap(base + m.off, m.len);
        a.MemRelease((CUmemGenericAllocationHandle)m.handle);
    }
    maps.clear();
    a.MemAddressFree(base, region_bytes * mapped_end.size());
    base = 0;
    mapped_end.clear();
}

// ------------------------------------------------------------------ host plan
// Chunks: consecutive ranges of the shard's clusters on the top active level l0, balanced by
// the number of row pairs below them; G is clamped to the number of those clusters.
void lean_plan(Shard* C, int G) {
    Structure& S = C->st;
    const ClusterTree& T = S.ct;
    const int L = T.depth, k = C->k, me = C->rank;
    PassH& X = C->row;
    LeanState& Ln = C->lean;
    if (!C->sym_ok) throw NotImpl("the memory-lean plan needs the adjoint-symmetric structure (" + C->sym_why + ")");
    Ln.clear_plan();
    int l0 = -1;
    for (int l = 0; l <= L && l0 < 0; ++l)
        if (X.own_hi[l] > X.own_lo[l]) l0 = l;
    if (l0 < 0) throw NotImpl("no row pairs on this shard");
    Ln.l0 = l0;
    // top clusters of this shard on level l0 and their pair weights
    std::vector<int64_t> tops;
    for (int64_t t : T.levels[l0])
        if (C->owner[t] == me) tops.push_back(t);
    const int ntop = (int)tops.size();
    G = std::max(1, std::min(G, ntop));
    Ln.G = G;
    std::vector<int> top_of(T.begin.size(), -1);  // cluster -> index of its l0 ancestor in tops
    for (int i = 0; i < ntop; ++i) top_of[tops[i]] = i;
    for (int l = l0 + 1; l <= L; ++l)
        for (int64_t t : T.levels[l]) top_of[t] = top_of[T.parent[t]];
    std::vector<double> wt(ntop, 0.0);
    for (int l = l0; l <= L; ++l)
        for (int p = X.own_lo[l]; p < X.own_hi[l]; ++p) wt[top_of[C->bp_t[X.bp[p]]]] += 1.0;
    // chunk g takes the top clusters whose weight midpoint falls in the g-th G-quantile
    std::vector<int> chunk_of_top(ntop, 0);
    {
        const double tot = std::max(1.0, std::accumulate(wt.begin(), wt.end(), 0.0));
        double acc = 0.0;
        for (int i = 0; i < ntop; ++i) {
            chunk_of_top[i] = std::min(G - 1, (int)(G * (acc + 0.5 * wt[i]) / tot));
            acc += wt[i];
        }
    }
    auto chunk_of = [&](int64_t t) { return top_of[t] < 0 ? -1 : chunk_of_top[top_of[t]]; };
    // row pairs per (g, l): contiguous (pairs of a level sorted by cluster, clusters BFS-numbered)
    Ln.p_lo.assign((size_t)G * (L + 1), 0);
    Ln.p_hi.assign((size_t)G * (L + 1), 0);
    for (int l = 0; l <= L; ++l) {
        for (int g = 0; g < G; ++g) Ln.p_lo[g * (L + 1) + l] = Ln.p_hi[g * (L + 1) + l] = X.own_lo[l];
        int p = X.own_lo[l];
        for (int g = 0; g < G; ++g) {
            Ln.p_lo[g * (L + 1) + l] = p;
            while (p < X.own_hi[l] && chunk_of(C->bp_t[X.bp[p]]) == g) ++p;
            Ln.p_hi[g * (L + 1) + l] = p;
        }
        if (p != X.own_hi[l]) throw std::logic_error("lean plan: chunk pairs not contiguous");
    }
    // blocks per chunk, slots
    std::vector<std::vector<int>> cb(G);
    for (int b = C->b_lo; b < C->b_hi; ++b) cb[chunk_of(C->blk_t[b])].push_back(b);
    Ln.blk_ptr.assign(G + 1, 0);
    std::vector<int> slot(C->st.blocks.size(), 0);
    for (int g = 0; g < G; ++g) {
        Ln.blk_ptr[g + 1] = Ln.blk_ptr[g] + (int)cb[g].size();
        for (size_t i = 0; i < cb[g].size(); ++i) {
            Ln.blk.push_back(cb[g][i]);
            slot[cb[g][i]] = (int)i;
        }
        Ln.S_slots = std::max<int64_t>(Ln.S_slots, (int64_t)cb[g].size());
    }
    C->lean_slot.swap(slot);
    // mirror reads only within the chunk's S slots
    C->lean_mirror.assign(C->st.blocks.size(), -1);
    for (int b = C->b_lo; b < C->b_hi; ++b) {
        const int mb = C->blk_mirror[b];
        if (mb >= C->b_lo && mb < C->b_hi && chunk_of(C->blk_t[mb]) == chunk_of(C->blk_t[b])) C->lean_mirror[b] = mb;
    }
    // direct (persistent) row basis pairs and row pairs
    const int nbp = (int)C->bp_t.size();
    Ln.keep.assign(nbp, 0);
    Ln.keepC.assign(X.bp.size(), 0);
    for (int b = C->b_lo; b < C->b_hi; ++b) {
        Ln.keep[C->blk_bprow[b]] = 1;
        Ln.keep[C->blk_bpcs[b]] = 1;
        Ln.keepC[C->blk_prow[b]] = 1;
        if (C->owner[C->blk_s[b]] == me) Ln.keepC[C->col2row[C->blk_pcol[b]]] = 1;
    }
    // the own row pairs that other shards' blocks reference through their column side: C exported
    for (int peer = 0; peer < C->world; ++peer)
        for (int p : C->C_send[peer]) Ln.keepC[C->col2row[p]] = 1;
    // (s,-c) of a block whose column cluster another shard owns: imported after phase b (R by QR,
    // exchange X_R) or regenerated here (leaf with #s <= k: R = V); its C' is imported after the
    // truncation into a slot of the C pool (lean_columns)
    auto r_by_qr = [&](int id) { return !T.is_leaf(C->bp_t[id]) || T.size(C->bp_t[id]) > k; };
    // VR layout: persistent slabs first, then per-chunk scratch (same offsets reused by every chunk)
    std::fill(C->bp_V_off.begin(), C->bp_V_off.end(), -1);
    std::fill(C->bp_R_off.begin(), C->bp_R_off.end(), -1);
    int64_t off = 0;
    for (int id = 0; id < nbp; ++id) {
        if (!Ln.keep[id]) continue;
        const int t = C->bp_t[id];
        if (!r_by_qr(id)) {
            C->bp_V_off[id] = C->bp_R_off[id] = off;
            off += T.size(t) * k;
        } else {
            C->bp_R_off[id] = off;
            off += (int64_t)C->bp_R_rows[id] * k;
        }
    }
    Ln.VR_persist = off;
    Ln.lvi.clear();
    for (int id = 0; id < nbp; ++id)
        if (Ln.keep[id] && !C->bp_own[id] && !r_by_qr(id)) Ln.lvi.push_back(id);
    Ln.qr_ptr.assign((size_t)G * (L + 1) + 1, 0);
    Ln.lvb_ptr.assign((size_t)G * (L + 1) + 1, 0);
    Ln.lvd_ptr.assign((size_t)G * (L + 1) + 1, 0);
    for (int g = 0; g < G; ++g) {
        int64_t cur = Ln.VR_persist;
        for (int l = 0; l <= L; ++l) {
            const int gl = g * (L + 1) + l;
            for (int p = Ln.p_lo[gl]; p < Ln.p_hi[gl]; ++p) {
                const int id = X.bp[p];
                const int t = C->bp_t[id];
                if (T.is_leaf(t)) {
                    Ln.lvb.push_back(id);
                    if (C->bp_V_off[id] < 0) {  // V in scratch (non-direct, or #t > k)
                        C->bp_V_off[id] = cur;
                        cur += T.size(t) * k;
                        Ln.lvd.push_back(id);
                        if (!r_by_qr(id)) C->bp_R_off[id] = C->bp_V_off[id];
                    }
                }
                if (r_by_qr(id)) {
                    Ln.qr.push_back(id);
                    if (C->bp_R_off[id] < 0) {
                        C->bp_R_off[id] = cur;
                        cur += (int64_t)C->bp_R_rows[id] * k;
                    }
                }
            }
            Ln.qr_ptr[gl + 1] = (int)Ln.qr.size();
            Ln.lvb_ptr[gl + 1] = (int)Ln.lvb.size();
            Ln.lvd_ptr[gl + 1] = (int)Ln.lvd.size();
        }
        Ln.VR_scratch = std::max(Ln.VR_scratch, cur - Ln.VR_persist);
    }
    C->VR_total = Ln.VR_persist + Ln.VR_scratch;
    // transfer factors of the row basis pairs only
    Ln.E_off.assign(nbp, -1);
    int64_t eoff = 0;
    for (int p = 0; p < (int)X.bp.size(); ++p) {
        const int id = X.bp[p];
        if (C->bp_own[id] && C->bp_child0[id] >= 0) {
            Ln.E_off[id] = eoff;
            eoff += 6LL * C->m * C->m;
        }
    }
    C->bp_E_off = Ln.E_off;
    C->E_total = Ln.E_total = eoff;
    // Zhat scratch per chunk (same offsets for every chunk)
    std::fill(X.Z_off.begin(), X.Z_off.end(), -1);
    for (int g = 0; g < G; ++g) {
        int64_t cur = 0;
        for (int l = 0; l <= L; ++l) {
            const int gl = g * (L + 1) + l;
            for (int p = Ln.p_lo[gl]; p < Ln.p_hi[gl]; ++p) {
                X.Z_off[p] = cur;
                cur += (int64_t)X.Z_rows[p] * k;
            }
        }
        Ln.Z_scratch = std::max(Ln.Z_scratch, cur);
    }
    X.Z_total = Ln.Z_scratch;
    Ln.kb_cur = X.kb;
    Ln.rowsb_cur = X.rowsb;
    Ln.C_off_cur.assign(X.bp.size(), -1);
    Ln.Q_off_cur.assign(X.bp.size(), -1);
    Ln.on = true;
}

// Device bytes of the lean plan: static allocations + an estimate of the rank-dependent pools
// (ranks assumed min(bound, max(8, k/4))).
double lean_bytes(const Shard* C) {
    const LeanState& Ln = C->lean;
    const PassH& X = C->row;
    const int k = C->k;
    const ClusterTree& T = C->st.ct;
    const int L = T.depth;
    double b = 16.0 * ((double)C->VR_total + Ln.E_total + Ln.Z_scratch + Ln.S_slots * (double)k * k);
    b += 8.0 * X.sig_total + (double)C->n * 7 * 32 + (double)C->nclusters * sizeof(GridD);
    b += (double)cq_scratch_bytes_bound(k);
    b += 16.0 * (double)k * (X.bp.size() + C->col.bp.size()) + 16.0 * 4 * C->n;  // matvec xh, yh, x, y
    const double r_est = std::max(8.0, k / 8.0);  // ranks measured on C4q/C5q: mean 11-20 at k = 125
    double cb = 0, qb = 0, comp = 0, st = 0;
    for (int g = 0; g < Ln.G; ++g)
        for (int l = 0; l <= L; ++l) {
            const int gl = g * (L + 1) + l;
            double c1 = 0, q1 = 0;
            for (int p = Ln.p_lo[gl]; p < Ln.p_hi[gl]; ++p) {
                c1 += (double)X.kb[p] * k;
                q1 += (double)X.kb[p] * X.rowsb[p];
            }
            cb = std::max(cb, c1);
            qb = std::max(qb, q1);
        }
    for (size_t p = 0; p < X.bp.size(); ++p) {
        const double r = std::min<double>(X.kb[p], r_est);
        const int t = C->bp_t[X.bp[p]];
        comp += r * (X.child0[p] < 0 ? (double)T.size(t) : 2.0 * r) + (Ln.keepC.size() && Ln.keepC[p] ? r * k : 0.0);
    }
    for (int b2 = C->b_lo; b2 < C->b_hi; ++b2) st += r_est * r_est;
    // scratch of the wide split truncation (k_trunc_qr64 -> k_trunc_jepi64) for the largest
    // chunk-level launch (bounded by its inner-level form, which also keeps Vhat)
    int npmax = 0;
    for (int g = 0; g < Ln.G; ++g)
        for (int l = 0; l <= L; ++l) {
            const int gl = g * (L + 1) + l;
            npmax = std::max(npmax, Ln.p_hi[gl] - Ln.p_lo[gl]);
        }
    b += (double)trunc_split64_scratch_bytes(npmax, false, k);
    return b + 16.0 * (cb * 1.5 + qb + comp + st);
}

// ------------------------------------------------------------------ execution
namespace {

inline int gl_of(const Shard* C, int g, int l) { return g * (C->st.ct.depth + 1) + l; }

template <typename T>
void upload_slice(DevBuf<T>& d, const std::vector<T>& h, int p0, int np, cudaStream_t s) {
    if (np) CK(cudaMemcpyAsync(d.p + p0, h.data() + p0, np * sizeof(T), cudaMemcpyHostToDevice, s));
}

// copy descriptors -> k_copy_mat
struct CopyList {
    std::vector<int64_t> so, dof;
    std::vector<int> rows, cols, lds;
    void add(int64_t s, int64_t d, int r, int c, int ld) {
        if (r <= 0 || c <= 0) return;
        so.push_back(s);
        dof.push_back(d);
        rows.push_back(r);
        cols.push_back(c);
        lds.push_back(ld);
    }
    size_t size() const { return so.size(); }
};

void run_copies(Shard* C, CopyList& cl, double2* base, cudaStream_t s, double& bytes) {
    if (!cl.size()) return;
    LeanState& Ln = C->lean;
    const size_t n = cl.size();
    if (Ln.d_soff.n < n) {
        CK(cudaStreamSynchronize(s));
        const size_t cap = std::max(n, Ln.d_soff.n * 2);
        Ln.d_soff.alloc(cap);
        Ln.d_doff.alloc(cap);
        Ln.d_rows.alloc(cap);
        Ln.d_cols.alloc(cap);
        Ln.d_lds.alloc(cap);
    }
    // descriptors from pageable host memory: the copies are staged before return, so the host
    // vectors may be reused afterwards
    CK(cudaMemcpyAsync(Ln.d_soff.p, cl.so.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(Ln.d_doff.p, cl.dof.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(Ln.d_rows.p, cl.rows.data(), n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(Ln.d_cols.p, cl.cols.data(), n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(Ln.d_lds.p, cl.lds.data(), n * 4, cudaMemcpyHostToDevice, s));
    C->timed("compact", 1, [&] {
        launch_copy_mat(base, base, Ln.d_soff.p, Ln.d_doff.p, Ln.d_rows.p, Ln.d_cols.p, Ln.d_lds.p, (int)n, s);
    });
    for (size_t i = 0; i < n; ++i) bytes += 32.0 * cl.rows[i] * cl.cols[i];
    Ln.compact_items += (int64_t)n;
}

void set_chunk_blocks(Shard* C, int g) {
    LeanState& Ln = C->lean;
    C->P.S = Ln.d_Ss.p;
    (void)g;
}

}  // namespace

// Phase b (basis weights, Eq. 18) of every chunk, bottom-up within the chunk: leaf V of the chunk
// (persistent slabs for direct pairs, scratch otherwise), then the QR weights level by level.
void lean_basis(Shard* C) {
    LeanState& Ln = C->lean;
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int L = T.depth, k = C->k, m = C->m;
    if (!Ln.lvi.empty())  // (s,-c) of other shards with R = V: regenerated from the replicated mesh
        C->timed("setup_leafV", 1, [&] { launch_leafV(P, Ln.d_lvi.p, (int)Ln.lvi.size(), C->max_leaf, s); });
    for (int g = 0; g < Ln.G; ++g) {
        for (int l = L; l >= Ln.l0; --l) {
            const int gl = gl_of(C, g, l);
            const int nv = Ln.lvb_ptr[gl + 1] - Ln.lvb_ptr[gl];
            if (nv) {
                C->timed("setup_leafV", 1, [&] { launch_leafV(P, Ln.d_lvb.p + Ln.lvb_ptr[gl], nv, C->max_leaf, s); });
                double ent = 0;
                for (int i = Ln.lvb_ptr[gl]; i < Ln.lvb_ptr[gl + 1]; ++i) ent += (double)T.size(C->bp_t[Ln.lvb[i]]) * k;
                auto& st = C->kstat["setup_leafV"];
                st.flops += ent * 7 * 6;
                st.bytes += ent * 16 + ent / k * 7 * 32;
            }
        }
        for (int l = L; l >= Ln.l0; --l) {
            const int gl = gl_of(C, g, l);
            const int nb = Ln.qr_ptr[gl + 1] - Ln.qr_ptr[gl];
            if (!nb) continue;
            const std::string cls = "basis@" + std::to_string(l);
            C->timed(cls, 1, [&] { launch_basis(P, Ln.d_qr.p + Ln.qr_ptr[gl], nb, C->basis_maxrows[l], s); });
            double fl = 0;
            for (int i = Ln.qr_ptr[gl]; i < Ln.qr_ptr[gl + 1]; ++i) {
                const int id = Ln.qr[i];
                int rows;
                if (C->bp_child0[id] < 0)
                    rows = (int)T.size(C->bp_t[id]);
                else {
                    rows = C->bp_R_rows[C->bp_child0[id]] + C->bp_R_rows[C->bp_child1[id]];
                    fl += 8.0 * 3 * rows * k * m;
                }
                if (rows > k) {
                    const double M = rows, N = k, K = std::min(M, N);
                    fl += 16.0 * (M * N * K - (M + N) * K * K / 2.0 + K * K * K / 3.0);  // as qr_flops (dh2_api.cu)
                }
            }
            C->kstat[cls].flops += fl;
        }
    }
}

// Phases c-d of chunk g: leaf V regenerated, S_b of the chunk's blocks, block weights, total
// weights (top-down), truncation (bottom-up) with per-level compaction of Q/F and C.
void lean_chunk_weights_truncate(Shard* C, int g, double eps, int mode) {
    LeanState& Ln = C->lean;
    PlanD& P = C->P;
    PassH& X = C->row;
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int L = T.depth, k = C->k, m = C->m;
    // leaf V that is not persistent
    for (int l = L; l >= Ln.l0; --l) {
        const int gl = gl_of(C, g, l);
        const int nv = Ln.lvd_ptr[gl + 1] - Ln.lvd_ptr[gl];
        if (!nv) continue;
        C->timed("setup_leafV", 1, [&] { launch_leafV(P, Ln.d_lvd.p + Ln.lvd_ptr[gl], nv, C->max_leaf, s); });
        double ent = 0;
        for (int i = Ln.lvd_ptr[gl]; i < Ln.lvd_ptr[gl + 1]; ++i) ent += (double)T.size(C->bp_t[Ln.lvd[i]]) * k;
        auto& st = C->kstat["setup_leafV"];
        st.flops += ent * 7 * 6;
        st.bytes += ent * 16 + ent / k * 7 * 32;
    }
    // S_b of the chunk's blocks, block weights
    const int nb = Ln.blk_ptr[g + 1] - Ln.blk_ptr[g];
    const int* bl = Ln.d_blk.p + Ln.blk_ptr[g];
    set_chunk_blocks(C, g);
    if (nb) {
        C->timed("setup_S", 1, [&] { launch_S(P, 0, nb, s, bl); });
        auto& st = C->kstat["setup_S"];
        st.flops += (double)nb * k * k * 20;
        st.bytes += (double)nb * k * k * 16;
        C->timed("block_weights", 1, [&] { launch_block_weights(P, 0, nb, mode, Ln.d_mirror.p, s, bl); });
        double fl = 0;
        for (int i = Ln.blk_ptr[g]; i < Ln.blk_ptr[g + 1]; ++i) {
            const int b = Ln.blk[i];
            double rt = C->bp_R_rows[C->blk_bprow[b]], rs = C->bp_R_rows[C->blk_bpcs[b]];
            fl += 8.0 * (rt * k * k + rt * rs * k);
        }
        C->kstat["block_weights"].flops += fl;
    }
    // leaf levels whose total weights are folded into the truncation (fuse_leaf_weights)
    std::vector<char> fused(L + 1, 0);
    for (int l = Ln.l0; l <= L; ++l) {
        const int gl = gl_of(C, g, l);
        const int p0 = Ln.p_lo[gl], np = Ln.p_hi[gl] - p0;
        if (!np) continue;
        bool all_leaf = true;
        int rows = 0, mz = 0;
        for (int p = p0; p < p0 + np; ++p) {
            all_leaf = all_leaf && X.child0[p] < 0;
            rows = std::max(rows, (int)T.size(C->bp_t[X.bp[p]]));
            mz = std::max(mz, X.Z_rows[p]);
        }
        fused[l] = all_leaf && fuse_leaf_level(C, rows, mz, np);
        if (fused[l] && g == 0) C->fused_levels[0].push_back(l);
    }
    // total weights, top-down (Zhat of the chunk in the scratch slab)
    for (int l = Ln.l0; l <= L; ++l) {
        const int gl = gl_of(C, g, l);
        const int p0 = Ln.p_lo[gl], np = Ln.p_hi[gl] - p0;
        if (!np || fused[l]) continue;
        const std::string cls = "total_weights_row@" + std::to_string(l);
        bool all_leaf = true;
        for (int p = p0; p < p0 + np; ++p) all_leaf = all_leaf && X.child0[p] < 0;
        C->timed(cls, 1, [&] { launch_total_weights(P, true, p0, np, Ln.d_mirror.p, s, all_leaf); });
        double fl = 0;
        for (int p = p0; p < p0 + np; ++p) {
            for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) fl += 8.0 * C->bp_R_rows[C->blk_bpcs[X.blk[ib]]] * (double)k * k;
            for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) fl += 8.0 * 3 * X.Z_rows[X.par[ip]] * (double)k * m;
            if (X.total_rows[p] > k) fl += 8.0 * X.total_rows[p] * (double)k * k;
        }
        C->kstat[cls].flops += fl;
    }
    // truncation, bottom-up: bound layout in the scratch regions, then compaction
    int cbuf = 0;  // compact-scratch buffer of the level (regions 2 / 3 of the C pool alternate)
    for (int l = L; l >= Ln.l0; --l) {
        const int gl = gl_of(C, g, l);
        const int p0 = Ln.p_lo[gl], np = Ln.p_hi[gl] - p0;
        if (!np) continue;
        bool all_leaf = true, any_leaf = false;
        for (int p = p0; p < p0 + np; ++p) {
            all_leaf = all_leaf && X.child0[p] < 0;
            any_leaf = any_leaf || X.child0[p] < 0;
        }
        int maxrows = 0, maxz = 0;
        int64_t cc = 0, qc = 0;
        for (int p = p0; p < p0 + np; ++p) {
            const int rows = X.child0[p] < 0 ? (int)T.size(C->bp_t[X.bp[p]]) : X.rank[X.child0[p]] + X.rank[X.child1[p]];
            Ln.rowsb_cur[p] = rows;
            Ln.kb_cur[p] = std::min(rows, X.Z_rows[p]);
            Ln.C_off_cur[p] = Ln.Cpool.region_off(1) + cc;
            Ln.Q_off_cur[p] = qc + Ln.Qpool.region_off(1);
            cc += (int64_t)Ln.kb_cur[p] * k;
            qc += (int64_t)Ln.kb_cur[p] * rows;
            maxrows = std::max(maxrows, rows);
            maxz = std::max(maxz, X.Z_rows[p]);
        }
        Ln.Cpool.ensure(1, (size_t)cc * sizeof(double2));
        Ln.Qpool.ensure(1, (size_t)qc * sizeof(double2));
        upload_slice(X.d_kb, Ln.kb_cur, p0, np, s);
        upload_slice(X.d_rowsb, Ln.rowsb_cur, p0, np, s);
        upload_slice(X.d_C_off, Ln.C_off_cur, p0, np, s);
        upload_slice(X.d_Q_off, Ln.Q_off_cur, p0, np, s);
        truncate_level(C, X, true, l, p0, np, maxrows, maxz, all_leaf, fused[l] != 0, eps, mode, Ln.d_mirror.p);
        // compaction: Q/F -> persistent (ld = rows), C -> persistent (direct pairs) or the level's
        // compact scratch (read by the parent level only); ld = rank afterwards
        CopyList qlist, clist;
        int64_t scr = 0;
        const int creg = 2 + cbuf;
        for (int p = p0; p < p0 + np; ++p) {
            const int r = X.rank[p], rows = Ln.rowsb_cur[p];
            const int64_t qdst = Ln.Q_used;
            qlist.add(Ln.Q_off_cur[p], qdst, rows, r, rows);
            Ln.Q_used += (int64_t)rows * r;
            int64_t cdst;
            if (Ln.keepC[p]) {
                cdst = Ln.C_used;
                Ln.C_used += (int64_t)r * k;
            } else {
                cdst = Ln.Cpool.region_off(creg) + scr;
                scr += (int64_t)r * k;
            }
            clist.add(Ln.C_off_cur[p], cdst, r, k, Ln.kb_cur[p]);
            Ln.Q_off_cur[p] = qdst;
            Ln.C_off_cur[p] = cdst;
            Ln.kb_cur[p] = r;
        }
        Ln.Qpool.ensure(0, (size_t)Ln.Q_used * sizeof(double2));
        Ln.Cpool.ensure(0, (size_t)Ln.C_used * sizeof(double2));
        Ln.Cpool.ensure(creg, (size_t)scr * sizeof(double2));
        double by = 0;
        run_copies(C, qlist, Ln.Qpool.ptr(), s, by);
        run_copies(C, clist, Ln.Cpool.ptr(), s, by);
        C->kstat["compact"].bytes += by;
        upload_slice(X.d_kb, Ln.kb_cur, p0, np, s);
        upload_slice(X.d_C_off, Ln.C_off_cur, p0, np, s);
        upload_slice(X.d_Q_off, Ln.Q_off_cur, p0, np, s);
        // the host vectors are rewritten by the next level: finish the uploads of this one first
        CK(cudaStreamSynchronize(s));
        cbuf ^= 1;
    }
}

void lean_alias_columns(Shard* C) {
    LeanState& Ln = C->lean;
    PassH &R = C->row, &X = C->col;
    cudaStream_t s = C->stream;
    const int np = (int)X.bp.size();
    std::vector<int> kb(np, 0), rowsb(np, 0);
    std::vector<char> own(np, 0);
    for (int l = 0; l < (int)X.own_lo.size(); ++l)
        for (int p = X.own_lo[l]; p < X.own_hi[l]; ++p) own[p] = 1;
    for (int p = 0; p < np; ++p) {
        const int q = C->col2row[p];
        X.C_off[p] = own[p] ? Ln.C_off_cur[q] : -1;
        X.Q_off[p] = own[p] ? Ln.Q_off_cur[q] : -1;
        kb[p] = own[p] ? Ln.kb_cur[q] : 0;
        rowsb[p] = own[p] ? Ln.rowsb_cur[q] : 0;
    }
    // C' of column pairs owned by other shards: compact slots (rank x k, ld rank) after the
    // persistent C, filled by the exchange X_C (ranks imported by X_RANK)
    for (int peer = 0; peer < C->world; ++peer)
        for (int p : C->C_recv[peer]) {
            X.C_off[p] = Ln.C_used;
            kb[p] = X.rank[p];
            Ln.C_used += (int64_t)X.rank[p] * C->k;
        }
    Ln.Cpool.ensure(0, (size_t)Ln.C_used * sizeof(double2));
    X.d_C_off.upload(X.C_off, s);
    X.d_Q_off.upload(X.Q_off, s);
    X.d_kb.upload(kb, s);
    X.d_rowsb.upload(rowsb, s);
    X.kb.swap(kb);  // host copies follow the device (exports); the column bounds are not used by the lean plan
    X.rowsb.swap(rowsb);
    C->P.col.C_off = X.d_C_off.p;
    C->P.col.Q_off = X.d_Q_off.p;
    C->P.col.kb = X.d_kb.p;
    C->P.col.rowsb = X.d_rowsb.p;
    C->P.col.C = C->P.row.C;
    C->P.col.Q = C->P.row.Q;
    (void)R;
    CK(cudaStreamSynchronize(s));
}

// Projection chunk by chunk with S_b regenerated; S~ laid out by the final ranks.
void lean_project(Shard* C) {
    LeanState& Ln = C->lean;
    PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const int k = C->k;
    const int nbt = (int)C->st.blocks.size();
    C->blk_St_off.assign(nbt, -1);
    C->St_total = 0;
    for (int b = C->b_lo; b < C->b_hi; ++b) {
        C->blk_St_off[b] = C->St_total;
        C->St_total += (int64_t)C->row.rank[C->blk_prow[b]] * C->col.rank[C->blk_pcol[b]];
    }
    CK(cudaStreamSynchronize(s));
    Ln.d_Zs.free();  // Zhat is dead: its memory goes to S~
    C->d_St.alloc(C->St_total);
    C->d_blk_St_off.upload(C->blk_St_off, s);
    P.St = C->d_St.p;
    P.blk_St_off = C->d_blk_St_off.p;
    for (int g = 0; g < Ln.G; ++g) {
        const int nb = Ln.blk_ptr[g + 1] - Ln.blk_ptr[g];
        if (!nb) continue;
        const int* bl = Ln.d_blk.p + Ln.blk_ptr[g];
        set_chunk_blocks(C, g);
        C->timed("setup_S", 1, [&] { launch_S(P, 0, nb, s, bl); });
        auto& st = C->kstat["setup_S"];
        st.flops += (double)nb * k * k * 20;
        st.bytes += (double)nb * k * k * 16;
        int maxkrow = 0;
        double fl = 0;
        for (int i = Ln.blk_ptr[g]; i < Ln.blk_ptr[g + 1]; ++i) {
            const int b = Ln.blk[i];
            const double kt = C->row.rank[C->blk_prow[b]], ks = C->col.rank[C->blk_pcol[b]];
            maxkrow = std::max(maxkrow, (int)kt);
            fl += 8.0 * (kt * k * k + kt * ks * k);
        }
        C->timed("project", 1, [&] { launch_project(P, 0, nb, maxkrow, Ln.d_mirror.p, s, bl); });
        C->kstat["project"].flops += fl;
    }
}

// Device allocations of the lean plan that upload_all does not make (pools of rank-dependent
// size; the Zhat scratch), and the lean versions of the tables upload_all uploaded.
void lean_alloc(Shard* C) {
    LeanState& Ln = C->lean;
    PlanD& P = C->P;
    cudaStream_t s = C->stream;
    size_t freeb = 0, totb = 0;
    CK(cudaMemGetInfo(&freeb, &totb));
    Ln.Cpool.reserve(C->device, 4, totb);
    Ln.Qpool.reserve(C->device, 2, totb);
    P.row.C = Ln.Cpool.ptr();
    P.row.Q = Ln.Qpool.ptr();
    P.col.C = P.row.C;
    P.col.Q = P.row.Q;
    Ln.d_blk.upload(Ln.blk, s);
    Ln.d_qr.upload(Ln.qr, s);
    Ln.d_lvb.upload(Ln.lvb, s);
    Ln.d_lvd.upload(Ln.lvd, s);
    Ln.d_lvi.upload(Ln.lvi, s);
    Ln.d_mirror.upload(C->lean_mirror, s);
    C->d_blk_slot.upload(C->lean_slot, s);
    P.blk_slot = C->d_blk_slot.p;
    Ln.d_Ss.alloc((size_t)Ln.S_slots * C->k * C->k);
    P.S = Ln.d_Ss.p;
    CK(cudaStreamSynchronize(s));
}

// Phases of the lean recompression; the context runs them shard by shard with the exchanges of
// SURVEY §8(e) in between (dh2_api.cu do_recompress): lean_begin, lean_basis [X_R],
// lean_weights_truncate [X_RANK], lean_columns [X_C], lean_project.
void lean_begin(Shard* C) {
    LeanState& Ln = C->lean;
    PassH& X = C->row;
    if (!(C->sym_ok && C->sym_opt)) throw NotImpl("the memory-lean plan needs adjoint_symmetry = 1");
    C->P.sym = 1;
    C->sym_used = true;
    C->fused_levels[0].clear();
    C->fused_levels[1].clear();
    C->fused_append = 0;
    Ln.C_used = Ln.Q_used = 0;
    Ln.compact_items = 0;
    if (!Ln.d_Zs.p && Ln.Z_scratch) Ln.d_Zs.alloc(Ln.Z_scratch);
    C->P.row.Z = Ln.d_Zs.p;
    // the Zhat offsets are the chunk-relative lean ones
    X.d_Z_off.upload(X.Z_off, C->stream);
    C->P.row.Z_off = X.d_Z_off.p;
}

void lean_weights_truncate(Shard* C, double eps, int mode) {
    LeanState& Ln = C->lean;
    PassH& X = C->row;
    const int L = C->st.ct.depth;
    X.rank.assign(X.bp.size(), 0);
    for (int g = 0; g < Ln.G; ++g) lean_chunk_weights_truncate(C, g, eps, mode);
    // column pass by the adjoint symmetry (ranks mirrored; factors read conjugated)
    PassH& Y = C->col;
    Y.rank.assign(Y.bp.size(), 0);
    for (int l = 0; l <= L; ++l) {
        const int p0 = Y.own_lo[l], np = Y.own_hi[l] - p0;
        if (!np) continue;
        C->timed("mirror_col", 1, [&] { launch_mirror_pass(C->P, C->d_col2row.p, p0, np, C->stream); });
        for (int p = p0; p < p0 + np; ++p) Y.rank[p] = X.rank[C->col2row[p]];
    }
}

void lean_columns(Shard* C) {
    PassH& Y = C->col;
    if (C->world > 1) {  // ranks of the imported column pairs (X_RANK) for their C' slots
        CK(cudaStreamSynchronize(C->stream));
        std::vector<int> all(Y.bp.size());
        CK(cudaMemcpy(all.data(), Y.d_rank.p, all.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int peer = 0; peer < C->world; ++peer)
            for (int p : C->C_recv[peer]) Y.rank[p] = all[p];
    }
    lean_alias_columns(C);
}

void lean_finish(Shard* C) {
    size_t freeb = 0, totb = 0;
    cudaMemGetInfo(&freeb, &totb);
    C->lean.peak_bytes = std::max(C->lean.peak_bytes, (double)(totb - freeb));
}

}  // namespace dh2
