// Multi-GPU plumbing of the C ABI: communicators (NCCL loaded at run time, or host
// callbacks supplied by the caller), and the time-sharded FD preconditioner / system operator.
//
// One process per GPU.  Rank r owns time slices T_r of every vector.  The FD apply transposes twice
// (time slabs -> spatial slabs for the time direction, and back); both transposes are fused into the
// epilogue of the producing stage kernel, which stores every output element straight into the owner
// rank's receive buffer (NVLink P2P stores through CUDA IPC pointers).  A stream-ordered barrier
// (a 1-element NCCL all-reduce) separates the stages.  The system mat-vec needs only the p edge slices
// of the time neighbours (banded time factors), pushed by peer copies into halo-extended buffers.
// The reference is serial: there is no reference counterpart to cite for this file.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'ed (the process may already hold torch's NCCL)

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "handles.hpp"

using namespace stiga;
using namespace stiga::capi;

namespace stiga {
stiga_fd_s* fd_build(int d, const int* n, const double* const* K, const double* const* M, int n_t, const double* Wt,
                     const double* Mt, double gamma, double nu, const double* scaling, long long scaling_len,
                     int device, const std::function<void(stiga_fd_s&)>& prepare, int flags,
                     const double* d_scaling);  // capi.cpp
stiga_kronsum_s* ks_build_spacetime(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                                    const double* Wt, const double* Mt, double gamma, double nu, int device);
stiga_kronsum_s* ks_build_physical(stiga_problem_s* prob, int p, int n_el, int device);
}  // namespace stiga

// ------------------------------------------------------------------------------------------
// NCCL, resolved at run time
// ------------------------------------------------------------------------------------------
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("NCCL not available: ") + dlerror();
            return a;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllReduce || !a.AllGather || !a.GetErrorString)
            a.error = "NCCL library lacks a required symbol";
        return a;
    }();
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaFailure(std::string(what) + ": " + nccl().GetErrorString(r));
}

const NcclApi& nccl_or_throw() {
    const NcclApi& a = nccl();
    if (!a.error.empty()) throw CudaFailure(a.error);
    return a;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// Communicator
// ------------------------------------------------------------------------------------------
struct stiga_comm_s {
    int world = 1, rank = 0, device = 0;
    int kind = 0;  // 0 = NCCL, 1 = host callbacks
    ncclComm_t nc = nullptr;
    stiga_comm_callbacks cb{};
    DBuf flag, tmp;

    ~stiga_comm_s() {
        if (nc) nccl().CommDestroy(nc);
    }
    void cbck(int status, const char* what) const {
        if (status != 0) throw CudaFailure(std::string("communicator callback ") + what + " failed (" +
                                           std::to_string(status) + ")");
    }
    // Stream-ordered barrier: kernels enqueued after it start only after every rank's stream reached it.
    void barrier(cudaStream_t st) {
        if (world == 1) return;
        if (kind == 0) {
            nck(nccl().AllReduce(flag.p, flag.p, 1, ncclDouble, ncclSum, nc, st), "barrier (ncclAllReduce)");
        } else {
            ck(cudaStreamSynchronize(st), "barrier sync");
            cbck(cb.barrier(cb.ctx), "barrier");
        }
    }
    void allreduce_dev(double* d, long long n, cudaStream_t st) {
        if (world == 1 || n == 0) return;
        if (kind == 0) {
            nck(nccl().AllReduce(d, d, static_cast<size_t>(n), ncclDouble, ncclSum, nc, st), "ncclAllReduce");
            return;
        }
        std::vector<double> h(n);
        ck(cudaMemcpyAsync(h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "allreduce D2H");
        ck(cudaStreamSynchronize(st), "allreduce sync");
        cbck(cb.allreduce(cb.ctx, h.data(), static_cast<int>(n), 0), "allreduce");
        ck(cudaMemcpyAsync(d, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "allreduce H2D");
        ck(cudaStreamSynchronize(st), "allreduce sync");
    }
    // Blocking all-gather of host bytes (setup only: IPC handles, partition checks).
    void allgather_host(const void* send, int bytes, void* recv) {
        if (world == 1) {
            std::memcpy(recv, send, bytes);
            return;
        }
        if (kind == 1) {
            cbck(cb.allgather(cb.ctx, send, bytes, recv), "allgather");
            return;
        }
        const size_t words = (static_cast<size_t>(bytes) + 7) / 8;
        tmp.ensure(words * (world + 1));
        ck(cudaMemset(tmp.p, 0, sizeof(double) * words * (world + 1)), "memset");
        ck(cudaMemcpy(tmp.p, send, bytes, cudaMemcpyHostToDevice), "allgather H2D");
        nck(nccl().AllGather(tmp.p, tmp.p + words, words, ncclDouble, nc, nullptr), "ncclAllGather");
        ck(cudaStreamSynchronize(nullptr), "allgather sync");
        std::vector<double> h(words * world);
        ck(cudaMemcpy(h.data(), tmp.p + words, sizeof(double) * words * world, cudaMemcpyDeviceToHost), "allgather D2H");
        for (int q = 0; q < world; ++q)
            std::memcpy(static_cast<char*>(recv) + static_cast<size_t>(q) * bytes, h.data() + q * words, bytes);
    }
};

namespace stiga {
void comm_allreduce(stiga_comm_s* C, double* d_buf, long long n, cudaStream_t st) { C->allreduce_dev(d_buf, n, st); }

Shard::~Shard() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
}
KronShard::~KronShard() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
}
}  // namespace stiga

namespace {

// Exchanges CUDA IPC handles of this rank's buffers and opens the peers' (peer access enabled
// lazily); ptrs[b][q] = buffer b of rank q as seen from this process (own buffers as is).
void exchange_buffers(stiga_comm_s& C, const std::vector<double*>& mine, std::vector<std::vector<double*>>& ptrs,
                      std::vector<void*>& opened) {
    const int nb = static_cast<int>(mine.size());
    std::vector<cudaIpcMemHandle_t> h(nb);
    for (int b = 0; b < nb; ++b) ck(cudaIpcGetMemHandle(&h[b], mine[b]), "cudaIpcGetMemHandle");
    std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(nb) * C.world);
    C.allgather_host(h.data(), static_cast<int>(sizeof(cudaIpcMemHandle_t) * nb), all.data());
    ptrs.assign(nb, std::vector<double*>(C.world, nullptr));
    for (int q = 0; q < C.world; ++q)
        for (int b = 0; b < nb; ++b) {
            if (q == C.rank) {
                ptrs[b][q] = mine[b];
                continue;
            }
            void* p = nullptr;
            ck(cudaIpcOpenMemHandle(&p, all[static_cast<size_t>(q) * nb + b], cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle");
            opened.push_back(p);
            ptrs[b][q] = static_cast<double*>(p);
        }
}

void check_comm(stiga_comm_s* C, const char* who) {
    require(C != nullptr, (std::string(who) + ": null communicator").c_str());
    require(C->world >= 1 && C->world <= STIGA_MAX_RANKS,
            (std::string(who) + ": world must be 1..STIGA_MAX_RANKS").c_str());
}

}  // namespace

// ------------------------------------------------------------------------------------------
// Sharded applies
// ------------------------------------------------------------------------------------------
namespace stiga {

void fd_apply_sharded(stiga_fd_s& P, const double* in, double* out, cudaStream_t st, std::vector<cudaEvent_t>* ev) {
    Shard& S = *P.shard;
    const int r = S.rank;
    P.prof_ev = ev;
    P.prof_i = 0;
    // space forward (D^-1/2 pre-scale + U_1^T..U_d^T), the last product scattering into the owners'
    // spatial-slab buffers; barrier; time stage on this rank's spatial slab scattering into the owners'
    // time-slab buffers; barrier; space backward with the D^-1/2 post-scale, local.
    P.apply_space_scatter(S.t_off[r], S.t_len[r], in, S.fwd, st);
    P.mark(st);
    S.comm->barrier(st);
    P.apply_time_scatter(S.s_off[r], S.s_len[r], S.slab_recv.p, S.tsc, st);
    P.mark(st);
    S.comm->barrier(st);
    P.apply_space(true, S.t_off[r], S.t_len[r], S.time_recv.p, out, st);
    P.mark(st);
    P.prof_ev = nullptr;
}

void kronsum_apply_sharded(stiga_kronsum_s& A, const double* x, double* y, cudaStream_t st) {
    KronShard& K = *A.kshard;
    const int r = K.rank, d = A.D - 1, nt = A.dims[d];
    const long long Ns = A.n_dof / nt;
    const long long ntl = K.t_len[r];
    // 1. every neighbour finished reading the halos it got from the previous apply
    K.comm->barrier(st);
    // 2. spatial halves of the local slab into the interior of the halo-extended buffers (fused path:
    //    for d = 3 the mode-(0,1) halves; mode 2 then runs inside the time stage, halos included)
    const bool fused = A.use_fused();
    if (fused) A.fused_space(ntl, x, K.ext_a.p + Ns * K.halo_lo, K.ext_b.p + Ns * K.halo_lo, st);
    else A.apply_space_slab(ntl, x, K.ext_a.p + Ns * K.halo_lo, K.ext_b.p + Ns * K.halo_lo, st);
    // 3. push the edge slices into the neighbours' halos (peer copies over NVLink)
    const size_t slab_bytes = sizeof(double) * static_cast<size_t>(Ns);
    if (K.prev_a) {  // my first slices -> previous rank's upper halo
        const int h = std::min<long long>(K.p, ntl);
        const long long dst = Ns * (K.prev_lo + K.prev_nt);
        ck(cudaMemcpyAsync(K.prev_a + dst, K.ext_a.p + Ns * K.halo_lo, slab_bytes * h, cudaMemcpyDeviceToDevice, st),
           "halo push");
        ck(cudaMemcpyAsync(K.prev_b + dst, K.ext_b.p + Ns * K.halo_lo, slab_bytes * h, cudaMemcpyDeviceToDevice, st),
           "halo push");
    }
    if (K.next_a) {  // my last slices -> next rank's lower halo
        const int h = K.next_lo;
        const long long src = Ns * (K.halo_lo + ntl - h);
        ck(cudaMemcpyAsync(K.next_a, K.ext_a.p + src, slab_bytes * h, cudaMemcpyDeviceToDevice, st), "halo push");
        ck(cudaMemcpyAsync(K.next_b, K.ext_b.p + src, slab_bytes * h, cudaMemcpyDeviceToDevice, st), "halo push");
    }
    // 4. the halos of this rank are complete once every rank passed the barrier
    K.comm->barrier(st);
    if (fused) {
        const int ti0 = static_cast<int>(K.t_off[r]) - K.halo_lo;
        A.fused_time(ti0, K.halo_lo + static_cast<int>(ntl) + K.halo_hi, static_cast<int>(K.t_off[r]), static_cast<int>(ntl),
                     K.ext_a.p, K.ext_b.p, y, st);
        return;
    }
    const int ia = A.physical ? 0 : 2 * d, ib = ia + 1;
    ck(gpu::launch_time_band_slab(Ns, nt, K.t_off[r], ntl, K.halo_lo, K.ext_a.p, K.ext_b.p, y, A.band(ia), A.band(ib),
                                  st),
       "time band slab");
}

}  // namespace stiga

namespace {

// Halo-extended buffers and neighbour pointers of a sharded system operator.
void attach_kshard(stiga_kronsum_s& A, stiga_comm_s* C) {
    const int d = A.D - 1, nt = A.dims[d];
    const long long Ns = A.n_dof / nt;
    auto K = std::make_unique<KronShard>();
    K->comm = C;
    K->world = C->world;
    K->rank = C->rank;
    partition(nt, C->world, K->t_off, K->t_len);
    const int ia = A.physical ? 0 : 2 * d, ib = ia + 1;
    K->p = std::max(A.hbw[ia], A.hbw[ib]);
    const int r = K->rank;
    require(*std::min_element(K->t_len.begin(), K->t_len.end()) >= std::max(1, C->world > 1 ? K->p : 1),
            "KronSumOperator (sharded): every rank needs at least p time slices (n_t >= p * world)");
    K->halo_lo = static_cast<int>(std::min<long long>(K->p, K->t_off[r]));
    K->halo_hi = static_cast<int>(std::min<long long>(K->p, nt - K->t_off[r] - K->t_len[r]));
    const long long ext = Ns * (K->halo_lo + K->t_len[r] + K->halo_hi);
    K->ext_a.alloc(static_cast<size_t>(ext));
    K->ext_b.alloc(static_cast<size_t>(ext));
    if (C->world > 1) {
        std::vector<std::vector<double*>> ptrs;
        exchange_buffers(*C, {K->ext_a.p, K->ext_b.p}, ptrs, K->opened);
        if (r > 0) {
            K->prev_a = ptrs[0][r - 1];
            K->prev_b = ptrs[1][r - 1];
            K->prev_lo = static_cast<int>(std::min<long long>(K->p, K->t_off[r - 1]));
            K->prev_nt = static_cast<int>(K->t_len[r - 1]);
        }
        if (r < C->world - 1) {
            K->next_a = ptrs[0][r + 1];
            K->next_b = ptrs[1][r + 1];
            K->next_lo = static_cast<int>(std::min<long long>(K->p, K->t_off[r + 1]));
        }
    }
    A.kshard = std::move(K);
}

}  // namespace

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
extern "C" {

int stiga_comm_unique_id(void* id_out) {
    return guarded([&] {
        require(id_out != nullptr, "stiga_comm_unique_id: null output");
        ncclUniqueId id;
        nck(nccl_or_throw().GetUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(ncclUniqueId) == STIGA_COMM_ID_BYTES, "NCCL unique id size");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int stiga_comm_init_nccl(int world, int rank, const void* id, int device, stiga_comm_t* out) {
    return guarded([&] {
        require(out && id, "stiga_comm_init_nccl: null argument");
        *out = nullptr;
        require(world >= 1 && world <= STIGA_MAX_RANKS && rank >= 0 && rank < world,
                "stiga_comm_init_nccl: world must be 1..STIGA_MAX_RANKS and 0 <= rank < world");
        const NcclApi& api = nccl_or_throw();
        DeviceGuard dg(device);
        auto C = std::make_unique<stiga_comm_s>();
        C->world = world;
        C->rank = rank;
        C->device = device;
        C->kind = 0;
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        nck(api.CommInitRank(&C->nc, world, uid, rank), "ncclCommInitRank");
        C->flag.alloc(1);
        ck(cudaMemset(C->flag.p, 0, sizeof(double)), "memset");
        *out = C.release();
    });
}

int stiga_comm_init_host(int world, int rank, const stiga_comm_callbacks* cb, int device, stiga_comm_t* out) {
    return guarded([&] {
        require(out && cb, "stiga_comm_init_host: null argument");
        *out = nullptr;
        require(world >= 1 && world <= STIGA_MAX_RANKS && rank >= 0 && rank < world,
                "stiga_comm_init_host: world must be 1..STIGA_MAX_RANKS and 0 <= rank < world");
        require(cb->allreduce && cb->allgather && cb->barrier, "stiga_comm_init_host: missing callback");
        auto C = std::make_unique<stiga_comm_s>();
        C->world = world;
        C->rank = rank;
        C->device = device;
        C->kind = 1;
        C->cb = *cb;
        *out = C.release();
    });
}

int stiga_comm_destroy(stiga_comm_t C) {
    return guarded([&] { delete C; });
}

int stiga_comm_info(stiga_comm_t C, int* world, int* rank, int* device, int* kind) {
    return guarded([&] {
        require(C != nullptr, "stiga_comm_info: null communicator");
        if (world) *world = C->world;
        if (rank) *rank = C->rank;
        if (device) *device = C->device;
        if (kind) *kind = C->kind;
    });
}

int stiga_comm_allreduce(stiga_comm_t C, double* d_buf, long long n, void* stream) {
    return guarded([&] {
        require(C && (n == 0 || d_buf) && n >= 0, "stiga_comm_allreduce: invalid argument");
        DeviceGuard dg(C->device);
        C->allreduce_dev(d_buf, n, as_stream(stream));
    });
}

int stiga_shard_partition(long long n, int world, int rank, long long* off, long long* len) {
    return guarded([&] {
        require(off && len, "stiga_shard_partition: null output");
        require(world >= 1 && rank >= 0 && rank < world && n >= 0, "stiga_shard_partition: invalid argument");
        std::vector<long long> o, l;
        partition(n, world, o, l);
        *off = o[rank];
        *len = l[rank];
    });
}

int stiga_fd_setup_sharded(int d, const int* n, const double* const* K, const double* const* M, int n_t,
                           const double* Wt, const double* Mt, double gamma, double nu, const double* scaling_local,
                           long long scaling_len, stiga_comm_t comm, stiga_fd_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_fd_setup_sharded: null handle output");
        *out = nullptr;
        check_comm(comm, "stiga_fd_setup_sharded");
        require(d >= 1 && n != nullptr && n_t >= 1, "ExtendedFDPreconditioner: per-direction matrices mismatch");
        long long n_s = 1;
        for (int l = 0; l < d; ++l) {
            require(n[l] >= 1, "spd_generalized_eig: shape mismatch");
            n_s *= n[l];
        }
        const int world = comm->world, rank = comm->rank;
        require(n_t >= world && n_s >= world,
                "ExtendedFDPreconditioner (sharded): fewer time slices or spatial indices than ranks");
        std::vector<long long> t_off, t_len, s_off, s_len;
        partition(n_t, world, t_off, t_len);
        partition(n_s, world, s_off, s_len);
        if (scaling_local) {
            require(scaling_len == n_s * t_len[rank], "ExtendedFDPreconditioner: scaling vector length mismatch");
            for (long long i = 0; i < scaling_len; ++i)
                require(scaling_local[i] > 0.0, "ExtendedFDPreconditioner: scaling must be strictly positive");
        }
        auto prepare = [&](stiga_fd_s& h) {
            auto S = std::make_unique<Shard>();
            S->comm = comm;
            S->world = world;
            S->rank = rank;
            S->t_off = t_off;
            S->t_len = t_len;
            S->s_off = s_off;
            S->s_len = s_len;
            h.nt_span = *std::max_element(t_len.begin(), t_len.end());
            h.ns_span = *std::max_element(s_len.begin(), s_len.end());
            h.scratch_len = std::max(n_s * h.nt_span, h.ns_span * n_t);
            if (scaling_local) {  // D^-1/2 of the slab (fdsolve.cpp:145-151), padded to nt_span slices for the tuner
                std::vector<double> dv(static_cast<size_t>(n_s * h.nt_span), 1.0);
                for (long long i = 0; i < scaling_len; ++i) dv[i] = 1.0 / std::sqrt(scaling_local[i]);
                h.dinv.upload(dv);
                h.dinv_t0 = t_off[rank];
            }
            S->slab_recv.alloc(static_cast<size_t>(s_len[rank] * n_t));
            S->time_recv.alloc(static_cast<size_t>(n_s * t_len[rank]));
            std::vector<std::vector<double*>> ptrs;
            if (world > 1) {
                exchange_buffers(*comm, {S->slab_recv.p, S->time_recv.p}, ptrs, S->opened);
            } else {
                ptrs = {{S->slab_recv.p}, {S->time_recv.p}};
            }
            // forward scatter: element (s, t) of the local time slab -> owner q of s, slab buffer
            // (|S_q| x n_t) at (s - s_off[q]) + |S_q| (t_off[r] + t)
            gpu::Scatter& F = S->fwd;
            F.G = world;
            F.by_time = 0;
            for (int q = 0; q < world; ++q) {
                F.off[q] = s_off[q];
                F.ld[q] = s_len[q];
                F.ptr[q] = ptrs[0][q];
                S->slab_ptr[q] = ptrs[0][q];
                S->time_ptr[q] = ptrs[1][q];
            }
            F.off[world] = n_s;
            F.a_shift = 0;
            F.b_shift = t_off[rank];
            // time scatter: element (s, t) of the local spatial slab -> owner q of t, time buffer
            // (N_s x |T_q|) at (s_off[r] + s) + N_s (t - t_off[q])
            gpu::Scatter& T = S->tsc;
            T.G = world;
            T.by_time = 1;
            for (int q = 0; q < world; ++q) {
                T.off[q] = t_off[q];
                T.ld[q] = n_s;
                T.ptr[q] = ptrs[1][q];
            }
            T.off[world] = n_t;
            T.a_shift = s_off[rank];
            T.b_shift = 0;
            h.shard = std::move(S);
        };
        *out = fd_build(d, n, K, M, n_t, Wt, Mt, gamma, nu, nullptr, 0, comm->device, prepare, 0, nullptr);
    });
}

int stiga_kronsum_create_spacetime_sharded(int d, const int* n, const double* const* K, const double* const* M,
                                           int n_t, const double* Wt, const double* Mt, double gamma, double nu,
                                           stiga_comm_t comm, stiga_kronsum_t* out) {
    return guarded([&] {
        require(out != nullptr, "stiga_kronsum_create_spacetime_sharded: null handle output");
        *out = nullptr;
        check_comm(comm, "stiga_kronsum_create_spacetime_sharded");
        std::unique_ptr<stiga_kronsum_s> A(ks_build_spacetime(d, n, K, M, n_t, Wt, Mt, gamma, nu, comm->device));
        DeviceGuard dg(comm->device);
        attach_kshard(*A, comm);
        *out = A.release();
    });
}

int stiga_kronsum_create_physical_sharded(stiga_problem_t prob, int p, int n_el, stiga_comm_t comm,
                                          stiga_kronsum_t* out) {
    return guarded([&] {
        require(out != nullptr && prob != nullptr, "stiga_kronsum_create_physical_sharded: null argument");
        *out = nullptr;
        check_comm(comm, "stiga_kronsum_create_physical_sharded");
        std::unique_ptr<stiga_kronsum_s> A(ks_build_physical(prob, p, n_el, comm->device));
        DeviceGuard dg(comm->device);
        attach_kshard(*A, comm);
        *out = A.release();
    });
}

}  // extern "C"
