// sharded.cu -- node-sharded sampling behind the C ABI (SURVEY 8(b) tgl_shard_create /
// tgl_sample_sharded, 8(e); row a12).  Not in the paper, which replicates the graph in host
// memory; here the T-CSR is split into node ranges over the ranks (graphs beyond one
// GPU's HBM), each rank building only its range (tgl_tcsr_build_range).
//
// One tgl_sample_sharded call runs Alg. 1's chains (layer 0 with its S snapshot blocks, then one
// chain per (layer, snapshot), R#3) and, per chain, the exchange protocol:
//
//   K8   bucket the chain's roots by owner range (stable: tgl_shard_bucket)
//   K7'  pack the requests (node, time, root key R#7, inherited lower bound R#3) in bucket order
//   X1   all-to-all of the per-peer request counts  -> host (sync 1)
//   X2   all-to-all-v of the requests
//   K4   the owner samples them on its range (sample_chain: the replicated mode's two kernels and
//        Philox counters, with the roots' own keys -> the replicated mode's bits)
//   X3   all-to-all of the per-peer reply edge counts -> host (sync 2)
//   X4   all-to-all-v of the replies: per-root counts + (nbr, eid, dt[, ts_edge]) per snapshot block
//   K8b  un-permute into the caller's blocks (original root order), then the next layer's root
//        keys (parent_key * k + j) and lower bounds are derived on the requesting rank
//
// X1..X4 are one grouped exchange each through a Transport: NCCL point-to-point (ncclSend /
// ncclRecv in one ncclGroupStart/End, over NVLink / NVSwitch) or, for tests on one device, an
// in-process group of ranks on threads exchanging with device copies.  NCCL is loaded with dlopen
// (the process's libnccl.so.2 -- torch's), so the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "chain.cuh"
#include "common.cuh"
#include "scan.cuh"

namespace tgl {

// ---------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

static NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv;
        return a;
    }();
    return api;
}

// ---------------------------------------------------------------------------- transports
// One grouped all-to-all-v: field f sends scnt[f][p] elements of elem[f] bytes, from send[f] at
// element offset prefix(scnt[f])[p], to peer p, and receives rcnt[f][p] elements into recv[f] at
// prefix(rcnt[f])[p].  Counts are host arrays.
struct Field {
    const void* send;
    void* recv;
    size_t elem;
    const int64_t* scnt;
    const int64_t* rcnt;
};

struct Transport {
    int rank = 0, world = 1;
    int64_t bytes_sent = 0, bytes_recv = 0;  // to / from OTHER ranks (NVLink traffic model)
    virtual ~Transport() {}
    virtual int exchange(const Field* f, int nf, cudaStream_t st) = 0;
    void count(const Field* f, int nf) {
        for (int q = 0; q < nf; ++q)
            for (int p = 0; p < world; ++p)
                if (p != rank) {
                    bytes_sent += f[q].scnt[p] * (int64_t)f[q].elem;
                    bytes_recv += f[q].rcnt[p] * (int64_t)f[q].elem;
                }
    }
};

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm) nccl().CommDestroy(comm);
    }
    int exchange(const Field* f, int nf, cudaStream_t st) override {
    NvtxRange nvtx_("exchange (NCCL)");
        NcclApi& A = nccl();
        count(f, nf);
        // this rank's own slice is a device-to-device copy on the stream (NCCL's send / recv to
        // self staged it through its channel buffers: the N = 1 C5 step moved ~1.2 GB that way)
        for (int q = 0; q < nf; ++q) {
            int64_t so = 0, ro = 0;
            for (int p = 0; p < rank; ++p) {
                so += f[q].scnt[p] * (int64_t)f[q].elem;
                ro += f[q].rcnt[p] * (int64_t)f[q].elem;
            }
            const size_t bytes = (size_t)f[q].scnt[rank] * f[q].elem;
            if (bytes && cudaMemcpyAsync(static_cast<char*>(f[q].recv) + ro, static_cast<const char*>(f[q].send) + so,
                                         bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return TGL_ECUDA;
        }
        if (world == 1) return TGL_OK;
        if (A.GroupStart() != ncclSuccess) return TGL_ENCCL;
        for (int q = 0; q < nf; ++q) {
            int64_t so = 0, ro = 0;
            for (int p = 0; p < world; ++p) {
                const size_t sb = (size_t)f[q].scnt[p] * f[q].elem, rb = (size_t)f[q].rcnt[p] * f[q].elem;
                if (p != rank) {
                    if (sb && A.Send(static_cast<const char*>(f[q].send) + so, sb, ncclUint8, p, comm, st) != ncclSuccess)
                        return A.GroupEnd(), TGL_ENCCL;
                    if (rb && A.Recv(static_cast<char*>(f[q].recv) + ro, rb, ncclUint8, p, comm, st) != ncclSuccess)
                        return A.GroupEnd(), TGL_ENCCL;
                }
                so += (int64_t)sb;
                ro += (int64_t)rb;
            }
        }
        return A.GroupEnd() == ncclSuccess ? TGL_OK : TGL_ENCCL;
    }
};

}  // namespace tgl

// In-process group (tests on one device): ranks are threads of one process; an exchange posts
// each rank's send pointers, then every rank copies its slices from its peers with cudaMemcpyAsync
// on its own stream, ordered after the senders' kernels by events.
struct tgl_shard_group {
    int world = 1;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    struct Post {
        std::vector<tgl::Field> f;
        cudaEvent_t ready = nullptr, done = nullptr;
    };
    std::vector<Post> post;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace tgl {

struct LocalTransport : Transport {
    tgl_shard_group* grp = nullptr;
    int exchange(const Field* f, int nf, cudaStream_t st) override {
        count(f, nf);
        auto& me = grp->post[rank];
        me.f.assign(f, f + nf);
        if (cudaEventRecord(me.ready, st) != cudaSuccess) return TGL_ECUDA;
        grp->barrier();  // every rank's send buffers are posted (and produced once `ready` fires)
        int rc = TGL_OK;
        for (int p = 0; p < world; ++p)  // every rank must post the same fields (else: no copies)
            if ((int)grp->post[p].f.size() != nf) rc = TGL_EINVAL;
        for (int p = 0; p < world && !rc; ++p) {
            auto& peer = grp->post[p];
            if (cudaStreamWaitEvent(st, peer.ready, 0) != cudaSuccess) rc = TGL_ECUDA;
            for (int q = 0; q < nf && !rc; ++q) {
                int64_t so = 0, ro = 0;  // peer's send offset to me, my receive offset from peer
                for (int r = 0; r < rank; ++r) so += peer.f[q].scnt[r];
                for (int r = 0; r < p; ++r) ro += f[q].rcnt[r];
                const size_t bytes = (size_t)f[q].rcnt[p] * f[q].elem;
                if (bytes && cudaMemcpyAsync(static_cast<char*>(f[q].recv) + ro * f[q].elem,
                                             static_cast<const char*>(peer.f[q].send) + so * f[q].elem, bytes,
                                             cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                    rc = TGL_ECUDA;
            }
        }
        if (!rc && cudaEventRecord(me.done, st) != cudaSuccess) rc = TGL_ECUDA;
        grp->barrier();  // every rank recorded `done` after its copies
        for (int p = 0; p < world && !rc; ++p)  // my send buffers stay untouched until peers copied
            if (cudaStreamWaitEvent(st, grp->post[p].done, 0) != cudaSuccess) rc = TGL_ECUDA;
        grp->barrier();  // nobody re-posts before every rank has waited on this round's events
        return rc;
    }
};

// ---------------------------------------------------------------------------- device buffers
// Grown on demand (first calls), reused afterwards; freed with the shard.
struct Buf {
    void* p = nullptr;
    size_t n = 0;
    template <typename T>
    T* get(size_t count, int* rc) {
        const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
        if (bytes > n) {
            if (p) cudaFree(p);
            p = nullptr;
            n = 0;
            if (cudaMalloc(&p, bytes + bytes / 4) != cudaSuccess) {
                *rc = TGL_ECUDA;
                return nullptr;
            }
            n = bytes + bytes / 4;
        }
        return static_cast<T*>(p);
    }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

__global__ void iota_keys_kernel(uint64_t base, int64_t n, uint64_t* __restrict__ key) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        key[i] = base + (uint64_t)i;
}

__global__ void pack_requests_kernel(const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ rn,
                                     const float* __restrict__ rt, const uint64_t* __restrict__ rk,
                                     const float* __restrict__ rlo, int32_t* __restrict__ qn, float* __restrict__ qt,
                                     uint64_t* __restrict__ qk, float* __restrict__ qlo) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = perm[j];
        qn[j] = rn[i];
        qt[j] = rt[i];
        qk[j] = rk[i];
        if (qlo) qlo[j] = rlo[i];
    }
}

// per-peer reply edge counts of every block: e[p * nsb + b] = edges of the roots received from p
__global__ void reply_counts_kernel(const int64_t* const* __restrict__ offs, int nsb, const int64_t* __restrict__ rcnt,
                                    int world, int64_t* __restrict__ e) {
    const int b = threadIdx.x;
    if (b >= nsb) return;
    int64_t r = 0;
    for (int p = 0; p < world; ++p) {
        const int64_t a = offs[b][r], z = offs[b][r + rcnt[p]];
        e[p * nsb + b] = z - a;
        r += rcnt[p];
    }
}

// next layer's roots of block b: key = parent_key * k + j (R#7), lower bound = the window's own
// (layer 0: t (-) (b+1) (x) t_s) or the inherited one (R#3)
__global__ void child_kernel(const int64_t* __restrict__ off, int64_t n, const uint64_t* __restrict__ rk,
                             const float* __restrict__ rt, const float* __restrict__ rlo, int layer, int b, float t_s,
                             int k, uint64_t* __restrict__ ck, float* __restrict__ clo) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = off[r], z = off[r + 1];
        const uint64_t key = rk[r] * (uint64_t)k;
        const float lo = clo ? (layer == 0 ? __fsub_rn(rt[r], __fmul_rn((float)(b + 1), t_s)) : rlo[r]) : 0.0f;
        for (int64_t o = a; o < z; ++o) {
            ck[o] = key + (uint64_t)(o - a);
            if (clo) clo[o] = lo;
        }
    }
}

__global__ void set_counts_kernel(int64_t* n_roots_dev, int64_t n, int64_t* nnz_dev, int64_t nnz) {
    *n_roots_dev = n;
    *nnz_dev = nnz;
}

}  // namespace tgl

struct tgl_shard {
    const tgl_tcsr* g = nullptr;
    int rank = 0, world = 1, device = 0;
    std::vector<int64_t> splits;
    tgl::Transport* tr = nullptr;
    int64_t host_syncs = 0;
    // buffers: splits, keys / lower bounds per (layer, snapshot) chain, bucketing, requests, local
    // blocks, replies, un-permute, counts
    tgl::Buf b_splits, b_key0, b_keys[2][TGL_MAX_SNAPSHOTS], b_lo[2][TGL_MAX_SNAPSHOTS], b_bucket, b_perm, b_cnt,
        b_qn, b_qt, b_qk, b_qlo, b_rn, b_rt, b_rk, b_rlo, b_chain, b_loff[TGL_MAX_SNAPSHOTS],
        b_lnbr[TGL_MAX_SNAPSHOTS], b_leid[TGL_MAX_SNAPSHOTS], b_ldt[TGL_MAX_SNAPSHOTS], b_lts[TGL_MAX_SNAPSHOTS],
        b_lcnt[TGL_MAX_SNAPSHOTS], b_scal, b_ecnt, b_offs, b_pcnt[TGL_MAX_SNAPSHOTS], b_pnbr[TGL_MAX_SNAPSHOTS],
        b_peid[TGL_MAX_SNAPSHOTS], b_pdt[TGL_MAX_SNAPSHOTS], b_pts[TGL_MAX_SNAPSHOTS], b_unperm;
    int64_t* h_cnt = nullptr;  // pinned host mirror of the count exchanges
    ~tgl_shard() {
        delete tr;
        if (h_cnt) cudaFreeHost(h_cnt);
    }
};

using namespace tgl;

extern "C" int tgl_shard_nccl_id(void* id) {
    if (!id) return TGL_EINVAL;
    NcclApi& A = nccl();
    if (!A.ok) return TGL_ENCCL;
    ncclUniqueId u;
    if (A.GetUniqueId(&u) != ncclSuccess) return TGL_ENCCL;
    static_assert(sizeof(ncclUniqueId) == TGL_NCCL_ID_BYTES, "ncclUniqueId size");
    memcpy(id, &u, sizeof(u));
    return TGL_OK;
}

extern "C" int tgl_shard_group_create(int32_t world, tgl_shard_group** out) {
    if (!out || world < 1 || world > 256) return TGL_EINVAL;
    tgl_shard_group* g = new tgl_shard_group;
    g->world = world;
    g->post.resize(world);
    for (auto& p : g->post)
        if (cudaEventCreateWithFlags(&p.ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming) != cudaSuccess) {
            delete g;
            return TGL_ECUDA;
        }
    *out = g;
    return TGL_OK;
}

extern "C" int tgl_shard_group_destroy(tgl_shard_group* g) {
    if (!g) return TGL_EINVAL;
    for (auto& p : g->post) {
        if (p.ready) cudaEventDestroy(p.ready);
        if (p.done) cudaEventDestroy(p.done);
    }
    delete g;
    return TGL_OK;
}

extern "C" int tgl_shard_create(const tgl_tcsr* local, const int64_t* splits, int32_t rank, int32_t world,
                                const void* nccl_id, tgl_shard_group* group, tgl_shard** out) {
    if (!out || !local || !splits || world < 1 || world > 256 || rank < 0 || rank >= world) return TGL_EINVAL;
    if ((nccl_id == nullptr) == (group == nullptr)) return TGL_EINVAL;  // exactly one transport
    if (group && group->world != world) return TGL_EINVAL;
    *out = nullptr;
    if (splits[0] != 0) return TGL_EINVAL;
    for (int r = 0; r < world; ++r)
        if (splits[r + 1] < splits[r]) return TGL_EINVAL;
    if (local->node_lo != splits[rank] || local->node_lo + local->n_nodes != splits[rank + 1]) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    tgl_shard* s = new tgl_shard;
    s->g = local;
    s->rank = rank;
    s->world = world;
    s->splits.assign(splits, splits + world + 1);
    cudaGetDevice(&s->device);
    if (cudaMallocHost(&s->h_cnt, sizeof(int64_t) * (2 + TGL_MAX_SNAPSHOTS) * 2 * 256) != cudaSuccess) {
        delete s;
        return TGL_ECUDA;
    }
    if (group) {
        LocalTransport* t = new LocalTransport;
        t->grp = group;
        s->tr = t;
    } else {
        NcclApi& A = nccl();
        if (!A.ok) {
            delete s;
            return TGL_ENCCL;
        }
        NcclTransport* t = new NcclTransport;
        ncclUniqueId u;
        memcpy(&u, nccl_id, sizeof(u));
        if (A.CommInitRank(&t->comm, world, u, rank) != ncclSuccess) {
            delete t;
            delete s;
            return TGL_ENCCL;
        }
        s->tr = t;
    }
    s->tr->rank = rank;
    s->tr->world = world;
    int64_t* sd = s->b_splits.get<int64_t>(world + 1, &rc);
    if (rc || cudaMemcpy(sd, splits, sizeof(int64_t) * (world + 1), cudaMemcpyHostToDevice) != cudaSuccess) {
        delete s;
        return TGL_ECUDA;
    }
    *out = s;
    return TGL_OK;
}

extern "C" int tgl_shard_destroy(tgl_shard* s) {
    if (!s) return TGL_EINVAL;
    delete s;
    return TGL_OK;
}

extern "C" int tgl_shard_stats(const tgl_shard* s, int64_t* bytes_sent, int64_t* bytes_recv, int64_t* host_syncs) {
    if (!s) return TGL_EINVAL;
    if (bytes_sent) *bytes_sent = s->tr->bytes_sent;
    if (bytes_recv) *bytes_recv = s->tr->bytes_recv;
    if (host_syncs) *host_syncs = s->host_syncs;
    return TGL_OK;
}

namespace tgl {

static unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

// one chain (layer l, snapshots [s0, s0 + nsb)) of the node-sharded protocol; outputs into out[b]
static int shard_chain(tgl_shard* sh, int l, int s0, int nsb, const int32_t* rn, const float* rt, const uint64_t* rk,
                       const float* rlo, int64_t n, int k, int strategy, float t_s, uint64_t seed, bool want_ts,
                       const tgl_block* const* out, int64_t* nnz_host, cudaStream_t st) {
    NvtxRange nvtx_("shard_chain");
    const int W = sh->world;
    int rc = TGL_OK;
    // K8: bucket by owner
    size_t bws = 0;
    if ((rc = tgl_shard_bucket_workspace(n, W, &bws))) return rc;
    void* bw = sh->b_bucket.get<char>(bws, &rc);
    int32_t* perm = sh->b_perm.get<int32_t>(std::max<int64_t>(n, 1), &rc);
    int64_t* cnt = sh->b_cnt.get<int64_t>(2 * 256 + 2 * 256 * TGL_MAX_SNAPSHOTS, &rc);  // send | recv | e_send | e_recv
    if (rc) return rc;
    int64_t* scnt_d = cnt;
    int64_t* rcnt_d = cnt + 256;
    int64_t* esend_d = cnt + 512;
    int64_t* erecv_d = esend_d + 256 * TGL_MAX_SNAPSHOTS;
    if ((rc = tgl_shard_bucket(rn, n, static_cast<const int64_t*>(sh->b_splits.p), W, perm, scnt_d, bw, bws, st)))
        return rc;
    // K7': requests in bucket order
    const bool has_lo = rlo != nullptr;
    int32_t* qn = sh->b_qn.get<int32_t>(n, &rc);
    float* qt = sh->b_qt.get<float>(n, &rc);
    uint64_t* qk = sh->b_qk.get<uint64_t>(n, &rc);
    float* qlo = has_lo ? sh->b_qlo.get<float>(n, &rc) : nullptr;
    if (rc) return rc;
    if (n > 0) pack_requests_kernel<<<grid_for(n), 256, 0, st>>>(perm, n, rn, rt, rk, rlo, qn, qt, qk, qlo);
    // X1: per-peer request counts
    std::vector<int64_t> ones(W, 1);
    {
        Field f{scnt_d, rcnt_d, sizeof(int64_t), ones.data(), ones.data()};
        if ((rc = sh->tr->exchange(&f, 1, st))) return rc;
    }
    int64_t* h = sh->h_cnt;
    if (cudaMemcpyAsync(h, cnt, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(h + 256, cnt + 256, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return TGL_ECUDA;
    ++sh->host_syncs;
    std::vector<int64_t> scnt(h, h + W), rcnt(h + 256, h + 256 + W);
    int64_t m = 0;  // roots this rank samples for the others
    for (int p = 0; p < W; ++p) m += rcnt[p];
    // X2: requests to their owners
    int32_t* qrn = sh->b_rn.get<int32_t>(m, &rc);
    float* qrt = sh->b_rt.get<float>(m, &rc);
    uint64_t* qrk = sh->b_rk.get<uint64_t>(m, &rc);
    float* qrlo = has_lo ? sh->b_rlo.get<float>(m, &rc) : nullptr;
    if (rc) return rc;
    {
        Field f[4] = {{qn, qrn, 4, scnt.data(), rcnt.data()},
                      {qt, qrt, 4, scnt.data(), rcnt.data()},
                      {qk, qrk, 8, scnt.data(), rcnt.data()},
                      {qlo, qrlo, 4, scnt.data(), rcnt.data()}};
        if ((rc = sh->tr->exchange(f, has_lo ? 4 : 3, st))) return rc;
    }
    // K4: sample the received roots on this rank's range
    ChainOut lo_out[TGL_MAX_SNAPSHOTS];
    int64_t* scal = sh->b_scal.get<int64_t>(2 * TGL_MAX_SNAPSHOTS, &rc);
    if (rc) return rc;
    for (int b = 0; b < nsb; ++b) {
        lo_out[b].offsets = sh->b_loff[b].get<int64_t>(m + 1, &rc);
        lo_out[b].nbr = sh->b_lnbr[b].get<int32_t>(m * k, &rc);
        lo_out[b].eid = sh->b_leid[b].get<int32_t>(m * k, &rc);
        lo_out[b].dt = sh->b_ldt[b].get<float>(m * k, &rc);
        lo_out[b].ts_edge = want_ts ? sh->b_lts[b].get<float>(m * k, &rc) : nullptr;
        lo_out[b].n_roots_dev = scal + 2 * b;
        lo_out[b].nnz_dev = scal + 2 * b + 1;
    }
    void* cw = sh->b_chain.get<char>(chain_workspace_bytes(m, nsb, k, strategy), &rc);
    if (rc) return rc;
    if ((rc = sample_chain(sh->g, l, s0, nsb, qrn, qrt, qrk, qrlo, m, k, strategy, t_s, seed, lo_out,
                           cw, sh->b_chain.n, st)))
        return rc;
    // per-root reply counts, per-peer reply edge counts
    int32_t* lcnt[TGL_MAX_SNAPSHOTS];
    const int64_t** offs = sh->b_offs.get<const int64_t*>(TGL_MAX_SNAPSHOTS, &rc);
    if (rc) return rc;
    const int64_t* offs_h[TGL_MAX_SNAPSHOTS];
    for (int b = 0; b < nsb; ++b) {
        lcnt[b] = sh->b_lcnt[b].get<int32_t>(m, &rc);
        if (rc) return rc;
        if ((rc = tgl_offsets_to_counts(lo_out[b].offsets, m, lcnt[b], st))) return rc;
        offs_h[b] = lo_out[b].offsets;
    }
    if (cudaMemcpyAsync(offs, offs_h, sizeof(offs_h[0]) * nsb, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return TGL_ECUDA;
    reply_counts_kernel<<<1, 32, 0, st>>>(offs, nsb, rcnt_d, W, esend_d);
    // X3: per-peer reply edge counts (nsb per peer)
    std::vector<int64_t> nsbv(W, nsb);
    {
        Field f{esend_d, erecv_d, sizeof(int64_t), nsbv.data(), nsbv.data()};
        if ((rc = sh->tr->exchange(&f, 1, st))) return rc;
    }
    if (cudaMemcpyAsync(h + 512, esend_d, sizeof(int64_t) * W * nsb, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(h + 512 + 256 * TGL_MAX_SNAPSHOTS, erecv_d, sizeof(int64_t) * W * nsb, cudaMemcpyDeviceToHost,
                        st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return TGL_ECUDA;
    ++sh->host_syncs;
    std::vector<int64_t> es((size_t)nsb * W), er((size_t)nsb * W);  // [b][p]
    int64_t tot[TGL_MAX_SNAPSHOTS] = {0};
    for (int p = 0; p < W; ++p)
        for (int b = 0; b < nsb; ++b) {
            es[(size_t)b * W + p] = h[512 + p * nsb + b];
            er[(size_t)b * W + p] = h[512 + 256 * TGL_MAX_SNAPSHOTS + p * nsb + b];
            tot[b] += er[(size_t)b * W + p];
        }
    // X4: replies (per block: counts over the requesters' roots, then the edges)
    std::vector<Field> f;
    int32_t* pcnt[TGL_MAX_SNAPSHOTS];
    int32_t* pnbr[TGL_MAX_SNAPSHOTS];
    int32_t* peid[TGL_MAX_SNAPSHOTS];
    float* pdt[TGL_MAX_SNAPSHOTS];
    float* pts[TGL_MAX_SNAPSHOTS];
    for (int b = 0; b < nsb; ++b) {
        pcnt[b] = sh->b_pcnt[b].get<int32_t>(n, &rc);
        pnbr[b] = sh->b_pnbr[b].get<int32_t>(tot[b], &rc);
        peid[b] = sh->b_peid[b].get<int32_t>(tot[b], &rc);
        pdt[b] = sh->b_pdt[b].get<float>(tot[b], &rc);
        pts[b] = want_ts ? sh->b_pts[b].get<float>(tot[b], &rc) : nullptr;
        if (rc) return rc;
        const int64_t* esb = es.data() + (size_t)b * W;
        const int64_t* erb = er.data() + (size_t)b * W;
        f.push_back({lcnt[b], pcnt[b], 4, rcnt.data(), scnt.data()});
        f.push_back({lo_out[b].nbr, pnbr[b], 4, esb, erb});
        f.push_back({lo_out[b].eid, peid[b], 4, esb, erb});
        f.push_back({lo_out[b].dt, pdt[b], 4, esb, erb});
        if (want_ts) f.push_back({lo_out[b].ts_edge, pts[b], 4, esb, erb});
    }
    if ((rc = sh->tr->exchange(f.data(), (int)f.size(), st))) return rc;
    // K8b: back to the original root order, into the caller's blocks
    void* uw = sh->b_unperm.get<char>(unpermute_workspace_bytes(n), &rc);
    if (rc) return rc;
    for (int b = 0; b < nsb; ++b) {
        const tgl_block& o = *out[b];
        if ((rc = unpermute_block(perm, n, pcnt[b], pnbr[b], peid[b], pdt[b], pts[b], o.offsets, o.nbr, o.eid, o.dt,
                                  want_ts ? o.ts_edge : nullptr, uw, sh->b_unperm.n, st)))
            return rc;
        set_counts_kernel<<<1, 1, 0, st>>>(o.n_roots_dev, n, o.nnz_dev, tot[b]);
        nnz_host[b] = tot[b];
    }
    return cudaGetLastError() == cudaSuccess ? TGL_OK : TGL_ECUDA;
}

}  // namespace tgl

extern "C" int tgl_sample_sharded(tgl_shard* sh, const int32_t* roots, const float* root_ts, int64_t n_roots,
                                  int32_t n_layers, const int32_t* fanouts, tgl_strategy strategy, int32_t n_snapshots,
                                  float snapshot_len, uint64_t seed, uint64_t root_key_base, tgl_block* out,
                                  void* stream) {
    NvtxRange nvtx_("tgl_sample_sharded");
    if (!sh || !out || !fanouts || n_roots < 0 || (n_roots > 0 && (!roots || !root_ts))) return TGL_EINVAL;
    const int L = n_layers, S = n_snapshots;
    int64_t roots_cap[64], edges_cap[64];
    size_t wsb = 0;
    int rc = tgl_sample_capacity(n_roots, L, fanouts, S, strategy, snapshot_len, roots_cap, edges_cap, &wsb);
    if (rc) return rc;
    if (n_roots >= (int64_t(1) << 31)) return TGL_EINVAL;
    for (int l = 0; l < L; ++l) {
        if (roots_cap[l] >= (int64_t(1) << 31)) return TGL_EINVAL;  // bucketing permutations are int32
        for (int s = 0; s < S; ++s) {
            const tgl_block& b = out[l * S + s];
            if (!b.offsets || !b.nbr || !b.eid || !b.dt || !b.n_roots_dev || !b.nnz_dev) return TGL_EINVAL;
            if (l < L - 1 && !b.ts_edge) return TGL_EINVAL;
            if (b.cap_roots < roots_cap[l] || b.cap_edges < edges_cap[l]) return TGL_ECAPACITY;
        }
    }
    rc = check_device();
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const bool finite = std::isfinite(snapshot_len);
    // layer 0: keys root_key_base + i, all S snapshot blocks in one chain
    uint64_t* k0 = sh->b_key0.get<uint64_t>(std::max<int64_t>(n_roots, 1), &rc);
    if (rc) return rc;
    if (n_roots > 0) iota_keys_kernel<<<grid_for(n_roots), 256, 0, st>>>(root_key_base, n_roots, k0);
    int64_t nnz[64][TGL_MAX_SNAPSHOTS];
    {
        const tgl_block* ob[TGL_MAX_SNAPSHOTS];
        bool ts0 = L > 1;  // ts_edge travels with the replies when a layer follows or the caller asked for it
        for (int s = 0; s < S; ++s) {
            ob[s] = &out[s];
            ts0 |= out[s].ts_edge != nullptr;
        }
        if ((rc = shard_chain(sh, 0, 0, S, roots, root_ts, k0, nullptr, n_roots, fanouts[0], strategy, snapshot_len,
                              seed, ts0, ob, nnz[0], st)))
            return rc;
    }
    // layer l >= 1: chain (l, s) over block (l-1, s)'s outputs (R#3, R#4), keys parent * k + j (R#7)
    const float* plo[TGL_MAX_SNAPSHOTS] = {nullptr};
    const uint64_t* pkey[TGL_MAX_SNAPSHOTS];
    const float* pts_[TGL_MAX_SNAPSHOTS];
    for (int s = 0; s < S; ++s) {
        pkey[s] = k0;
        pts_[s] = root_ts;
    }
    int64_t pn[TGL_MAX_SNAPSHOTS];
    for (int s = 0; s < S; ++s) pn[s] = n_roots;
    for (int l = 1; l < L; ++l) {
        for (int s = 0; s < S; ++s) {
            const tgl_block& par = out[(l - 1) * S + s];
            const int64_t m = nnz[l - 1][s];
            const int cur = l & 1;
            uint64_t* ck = sh->b_keys[cur][s].get<uint64_t>(std::max<int64_t>(m, 1), &rc);
            float* clo = finite ? sh->b_lo[cur][s].get<float>(std::max<int64_t>(m, 1), &rc) : nullptr;
            if (rc) return rc;
            if (pn[s] > 0)
                child_kernel<<<grid_for(pn[s]), 256, 0, st>>>(par.offsets, pn[s], pkey[s], pts_[s], plo[s], l - 1, s,
                                                              snapshot_len, fanouts[l - 1], ck, clo);
            const tgl_block* ob[1] = {&out[l * S + s]};
            if ((rc = shard_chain(sh, l, s, 1, par.nbr, par.ts_edge, ck, clo, m, fanouts[l], strategy, snapshot_len,
                                  seed, l < L - 1 || out[l * S + s].ts_edge != nullptr, ob, &nnz[l][s], st)))
                return rc;
            pkey[s] = ck;
            plo[s] = clo;
            pts_[s] = par.ts_edge;
            pn[s] = m;
        }
    }
    return TGL_OK;
}

// ---------------------------------------------------------------------------- sharded node state
// Node memory / mailbox sharded by the same node ranges (MAG's 121 M x (100 +
// K x 428) fp32 state does not fit one GPU -- the paper's APAN-on-MAG OOM).  Fig. 2 step
// 2 (gather) and step 6 (state write) across ranks, with the shard's transport:
//   gather       bucket the ids by owner (K8), X1 counts (sync), X2 ids, local tgl_gather on the
//                owner's rows, X3 rows back (sizes already known), request order restored through
//                the inverse permutation (tgl_perm_invert + tgl_gather);
//   state write  bucket the events by owner (stable: each owner receives them in (source rank,
//                batch index) order, the global event order of R#25), X1 counts (sync), X2 ids,
//                times and rows, local tgl_state_write on the owner's tables.
namespace tgl {

struct Route {
    int32_t* perm = nullptr;
    std::vector<int64_t> scnt, rcnt;
    int64_t m = 0;
};

static int route(tgl_shard* sh, const int32_t* ids, int64_t n, cudaStream_t st, Route& R) {
    const int W = sh->world;
    int rc = TGL_OK;
    size_t bws = 0;
    if ((rc = tgl_shard_bucket_workspace(n, W, &bws))) return rc;
    void* bw = sh->b_bucket.get<char>(bws, &rc);
    R.perm = sh->b_perm.get<int32_t>(std::max<int64_t>(n, 1), &rc);
    int64_t* cnt = sh->b_cnt.get<int64_t>(2 * 256 + 2 * 256 * TGL_MAX_SNAPSHOTS, &rc);
    if (rc) return rc;
    if ((rc = tgl_shard_bucket(ids, n, static_cast<const int64_t*>(sh->b_splits.p), W, R.perm, cnt, bw, bws, st)))
        return rc;
    std::vector<int64_t> ones(W, 1);
    Field f{cnt, cnt + 256, sizeof(int64_t), ones.data(), ones.data()};
    if ((rc = sh->tr->exchange(&f, 1, st))) return rc;
    int64_t* h = sh->h_cnt;
    if (cudaMemcpyAsync(h, cnt, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(h + 256, cnt + 256, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return TGL_ECUDA;
    ++sh->host_syncs;
    R.scnt.assign(h, h + W);
    R.rcnt.assign(h + 256, h + 256 + W);
    R.m = 0;
    for (int p = 0; p < W; ++p) R.m += R.rcnt[p];
    return TGL_OK;
}

}  // namespace tgl

extern "C" int tgl_shard_gather(tgl_shard* sh, const int32_t* ids, int64_t n, const tgl_gather_table* tables,
                                int32_t n_tables, void* stream) {
    NvtxRange nvtx_("tgl_shard_gather");
    if (!sh || n < 0 || (n > 0 && !ids) || n_tables < 1 || n_tables > TGL_MAX_GATHER_TABLES || !tables)
        return TGL_EINVAL;
    const int64_t lo = sh->splits[sh->rank], hi = sh->splits[sh->rank + 1];
    for (int j = 0; j < n_tables; ++j)
        if (tables[j].row_bytes <= 0 || tables[j].n_rows != hi - lo || (hi > lo && !tables[j].table) ||
            (n > 0 && !tables[j].out))
            return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Route R;
    if ((rc = route(sh, ids, n, st, R))) return rc;
    // X2: the ids to their owners (bucket order)
    int32_t* qids = sh->b_qn.get<int32_t>(n, &rc);
    int32_t* rids = sh->b_rn.get<int32_t>(R.m, &rc);
    if (rc) return rc;
    tgl_gather_table pk{ids, n, 4, qids};
    if (n > 0 && (rc = tgl_gather(R.perm, n, nullptr, &pk, 1, stream))) return rc;
    {
        Field f{qids, rids, 4, R.scnt.data(), R.rcnt.data()};
        if ((rc = sh->tr->exchange(&f, 1, st))) return rc;
    }
    // local rows (global ids: table bases offset by -lo rows), then X3 back to the requesters
    tgl_gather_table loc[TGL_MAX_GATHER_TABLES], back[TGL_MAX_GATHER_TABLES];
    Field f[TGL_MAX_GATHER_TABLES];
    for (int j = 0; j < n_tables; ++j) {
        const int64_t rb = tables[j].row_bytes;
        char* lrows = sh->b_lnbr[j].get<char>((size_t)std::max<int64_t>(R.m, 1) * rb, &rc);
        char* brows = sh->b_pnbr[j].get<char>((size_t)std::max<int64_t>(n, 1) * rb, &rc);
        if (rc) return rc;
        loc[j] = {static_cast<const char*>(tables[j].table) - lo * rb, hi, rb, lrows};
        back[j] = {brows, n, rb, tables[j].out};
        f[j] = {lrows, brows, (size_t)rb, R.rcnt.data(), R.scnt.data()};
    }
    if (R.m > 0 && (rc = tgl_gather(rids, R.m, nullptr, loc, n_tables, stream))) return rc;
    if ((rc = sh->tr->exchange(f, n_tables, st))) return rc;
    // request order: out[perm[j]] = back[j]  <=>  out[i] = back[inv[i]]
    int32_t* inv = sh->b_qk.get<int32_t>(std::max<int64_t>(n, 1), &rc);
    if (rc) return rc;
    if (n > 0 && ((rc = tgl_perm_invert(R.perm, n, inv, stream)) || (rc = tgl_gather(inv, n, nullptr, back, n_tables, stream))))
        return rc;
    return TGL_OK;
}

extern "C" int tgl_shard_state_write(tgl_shard* sh, const int32_t* ids, const float* ts, int64_t n, int32_t K,
                                     int32_t* pos, float* ts_table, const tgl_state_table* tables, int32_t n_tables,
                                     void* stream) {
    NvtxRange nvtx_("tgl_shard_state_write");
    // every rank exchanges the same fields (ids, times, rows): times are required whenever n > 0
    if (!sh || n < 0 || (n > 0 && (!ids || !ts)) || K < 1 || (K > 1 && !pos) || n_tables < 0 ||
        n_tables > TGL_MAX_GATHER_TABLES - 2 || (n_tables > 0 && !tables))
        return TGL_EINVAL;
    const int64_t lo = sh->splits[sh->rank], hi = sh->splits[sh->rank + 1];
    for (int j = 0; j < n_tables; ++j)
        if (tables[j].row_bytes <= 0 || (n > 0 && !tables[j].rows) || (hi > lo && !tables[j].table)) return TGL_EINVAL;
    int rc = check_device();
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Route R;
    if ((rc = route(sh, ids, n, st, R))) return rc;
    // pack (ids, times, rows) in bucket order, X2 to the owners
    const int nf = 2 + n_tables;
    tgl_gather_table pk[TGL_MAX_GATHER_TABLES];
    Field f[TGL_MAX_GATHER_TABLES];
    char* recv[TGL_MAX_GATHER_TABLES];
    int q = 0;
    auto add = [&](const void* src, int64_t rb) {
        char* packed = sh->b_pnbr[q].get<char>((size_t)std::max<int64_t>(n, 1) * rb, &rc);
        recv[q] = sh->b_lnbr[q].get<char>((size_t)std::max<int64_t>(R.m, 1) * rb, &rc);
        pk[q] = {src, n, rb, packed};
        f[q] = {packed, recv[q], (size_t)rb, R.scnt.data(), R.rcnt.data()};
        ++q;
    };
    add(ids, 4);
    add(ts, 4);
    for (int j = 0; j < n_tables; ++j) add(tables[j].rows, tables[j].row_bytes);
    if (rc) return rc;
    if (n > 0 && (rc = tgl_gather(R.perm, n, nullptr, pk, nf, stream))) return rc;
    if ((rc = sh->tr->exchange(f, nf, st))) return rc;
    // apply on the owner: global ids, local tables (bases offset by -lo nodes)
    tgl_state_table loc[TGL_MAX_GATHER_TABLES];
    for (int j = 0; j < n_tables; ++j)
        loc[j] = {recv[2 + j], tables[j].row_bytes,
                  static_cast<char*>(tables[j].table) - lo * (int64_t)K * tables[j].row_bytes};
    size_t wsb = 0;
    if ((rc = tgl_state_write_workspace(R.m, (int32_t)hi, &wsb))) return rc;
    void* ws = sh->b_unperm.get<char>(wsb, &rc);
    if (rc) return rc;
    return tgl_state_write(reinterpret_cast<const int32_t*>(recv[0]), reinterpret_cast<const float*>(recv[1]),
                           R.m, (int32_t)hi, K, pos ? pos - lo : nullptr, ts_table ? ts_table - lo * K : nullptr, loc,
                           n_tables, ws, wsb, stream);
}
