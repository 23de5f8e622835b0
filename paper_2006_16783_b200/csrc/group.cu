// Native multi-GPU group (include/txsite_b200.h "native multi-GPU group";
// DESIGN.md §6).  One process drives N contexts -- one per B200, or several on
// one device for testing -- as row-band shards of one grid:
// VIX / FINDMAX / VIEWSHED run per band with no exchange (one worker thread per
// rank, each stage call is synchronous on its own device), global candidate ids
// are the prefix of the band counts (block order), and the
// SITE rounds exchange one winner per round (commits stay
// serialized).  The device exchanges keep every round on the GPUs:
//   P2P   rank k: best key -> mailbox[k] = {key, payload} (own HBM), event;
//         rank j waits on every rank's event, its select kernel reads the N
//         keys and copies the winner's window rows out of the winner's mailbox
//         over NVLink (peer pointers), then applies it.  Mailboxes alternate by
//         round parity: round t+2's writer has passed round t+1's select, which
//         waited on every rank's round-t+1 export, which came after every rank's
//         round-t select -- so no reader of a mailbox can lag its next writer.
//   NCCL  one ncclAllGather of {key, payload} per round over ncclCommInitAll
//         communicators (distinct devices), then the same local select.
// Both are captured as one multi-device CUDA graph of kGraphRounds rounds and
// replayed until the device stop flag (decision D9, evaluated identically on
// every rank from the exchanged key) is set.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ctx.hpp"

namespace {

constexpr int kGraphRounds = 16;

// NCCL is opened on first use of TXS_XCHG_NCCL, not linked: a load-time
// dependency would bind the soname libnccl.so.2 to whichever copy loads first
// and break a torch imported later in the same process (torch ships its own,
// newer libnccl.so.2; when torch is already loaded, dlopen returns that copy).
struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi a;
    if (a.tried) return a;
    a.tried = true;
    // TXS_NCCL_LIB names a library explicitly; else a libnccl.so.2 already in the
    // process (torch's) is reused; else the system one is loaded
    void* h = nullptr;
    if (const char* e = getenv("TXS_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return a;
    a.CommInitAll = (decltype(a.CommInitAll))dlsym(h, "ncclCommInitAll");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.CommInitAll && a.CommDestroy && a.GroupStart && a.GroupEnd && a.AllGather && a.GetErrorString;
    return a;
}

const txs_engine_ops kDefaultOps = {
    txs_create, txs_destroy, txs_last_error, txs_set_shard, txs_shard_info, txs_set_terrain,
    txs_generate_fractal, txs_fill_rows, txs_estimate_vix, txs_find_candidates, txs_random_observers,
    txs_get_candidates, txs_set_candidate_base, txs_compute_viewsheds, txs_site_shard_begin,
    txs_site_shard_best, txs_site_shard_export, txs_site_shard_apply, txs_get_cumulative_rows, txs_get_stats,
};

}  // namespace

struct txs_group {
    txs_engine_ops ops{};
    bool native = true;                 // default ops: the device exchanges are available
    int n = 0;
    std::vector<int> dev;
    std::vector<txs_ctx*> ctx;
    std::string err;
    int32_t exchange = TXS_XCHG_REPLICATE;
    int64_t nrows = 0, ncols = 0, block = 0;
    int32_t roi = 0;
    std::vector<int64_t> r0, r1;
    int64_t observers = -1;             // >= 0 after txs_group_random_observers
    // device-round buffers (per rank, on its device)
    int64_t pw = 0;
    std::vector<uint64_t*> d_key, d_pay, d_gather, d_mail[2];
    std::vector<uint64_t**> d_peers[2];
    std::vector<cudaEvent_t> ev_mail[2], ev_join;
    cudaEvent_t ev_fork = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    std::vector<ncclComm_t> comms;
    bool peers_enabled = false;
    cudaGraphExec_t graph = nullptr;
    bool replicated = false;            // the last SITE ran on rank 0 over the gathered viewsheds
};

namespace {

txs_status gfail(txs_group* g, txs_status st, const std::string& msg) {
    g->err = msg;
    return st;
}

txs_status rank_fail(txs_group* g, int k, txs_status st) {
    g->err = "[rank " + std::to_string(k) + "] " + (g->ops.last_error ? g->ops.last_error(g->ctx[k]) : "error");
    return st;
}

txs_status cuda_gfail(txs_group* g, const char* what, cudaError_t e) {
    cudaGetLastError();
    return gfail(g, TXS_ERR_CUDA, std::string("[site] group ") + what + ": " + cudaGetErrorString(e));
}

#define G_CUDA(g, what, call)                                  \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return cuda_gfail(g, what, _e); \
    } while (0)

// fn(k) for every rank, one worker thread per rank (each stage call is
// synchronous on its own device, so the bands run concurrently)
template <class F>
txs_status for_ranks(txs_group* g, F&& fn) {
    std::vector<txs_status> st((size_t)g->n, TXS_OK);
    if (g->n == 1) {
        st[0] = fn(0);
    } else {
        std::vector<std::thread> th;
        th.reserve((size_t)g->n);
        for (int k = 0; k < g->n; ++k) th.emplace_back([&, k]() { st[(size_t)k] = fn(k); });
        for (auto& t : th) t.join();
    }
    for (int k = 0; k < g->n; ++k)
        if (st[(size_t)k] != TXS_OK) return rank_fail(g, k, st[(size_t)k]);
    return TXS_OK;
}

bool distinct_devices(const txs_group* g) {
    std::vector<int> d = g->dev;
    std::sort(d.begin(), d.end());
    return std::adjacent_find(d.begin(), d.end()) == d.end();
}

void free_round_buffers(txs_group* g) {
    if (g->graph) { cudaGraphExecDestroy(g->graph); g->graph = nullptr; }
    for (int k = 0; k < (int)g->d_key.size(); ++k) {
        cudaSetDevice(g->dev[(size_t)k]);
        for (uint64_t* p : {g->d_key[(size_t)k], g->d_pay[(size_t)k], g->d_gather[(size_t)k], g->d_mail[0][(size_t)k],
                            g->d_mail[1][(size_t)k]})
            if (p) cudaFree(p);
        for (int b = 0; b < 2; ++b)
            if (g->d_peers[b][(size_t)k]) cudaFree(g->d_peers[b][(size_t)k]);
    }
    g->d_key.clear(); g->d_pay.clear(); g->d_gather.clear();
    for (int b = 0; b < 2; ++b) { g->d_mail[b].clear(); g->d_peers[b].clear(); }
    g->pw = 0;
}

void destroy_events(txs_group* g) {
    for (int k = 0; k < (int)g->ev_join.size(); ++k) {
        cudaSetDevice(g->dev[(size_t)k]);
        for (int b = 0; b < 2; ++b) if (g->ev_mail[b][(size_t)k]) cudaEventDestroy(g->ev_mail[b][(size_t)k]);
        if (g->ev_join[(size_t)k]) cudaEventDestroy(g->ev_join[(size_t)k]);
    }
    g->ev_join.clear(); g->ev_mail[0].clear(); g->ev_mail[1].clear();
    if (!g->dev.empty()) cudaSetDevice(g->dev[0]);
    for (cudaEvent_t* e : {&g->ev_fork, &g->ev_t0, &g->ev_t1})
        if (*e) { cudaEventDestroy(*e); *e = nullptr; }
}

txs_status ensure_events(txs_group* g) {
    if (!g->ev_join.empty()) return TXS_OK;
    g->ev_join.assign((size_t)g->n, nullptr);
    g->ev_mail[0].assign((size_t)g->n, nullptr);
    g->ev_mail[1].assign((size_t)g->n, nullptr);
    for (int k = 0; k < g->n; ++k) {
        G_CUDA(g, "events", cudaSetDevice(g->dev[(size_t)k]));
        for (int b = 0; b < 2; ++b)
            G_CUDA(g, "events", cudaEventCreateWithFlags(&g->ev_mail[b][(size_t)k], cudaEventDisableTiming));
        G_CUDA(g, "events", cudaEventCreateWithFlags(&g->ev_join[(size_t)k], cudaEventDisableTiming));
    }
    G_CUDA(g, "events", cudaSetDevice(g->dev[0]));
    G_CUDA(g, "events", cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
    G_CUDA(g, "events", cudaEventCreate(&g->ev_t0));
    G_CUDA(g, "events", cudaEventCreate(&g->ev_t1));
    return TXS_OK;
}

txs_status enable_peers(txs_group* g) {
    if (g->peers_enabled) return TXS_OK;
    for (int i = 0; i < g->n; ++i)
        for (int j = 0; j < g->n; ++j) {
            const int a = g->dev[(size_t)i], b = g->dev[(size_t)j];
            if (a == b) continue;
            int ok = 0;
            G_CUDA(g, "peer access", cudaDeviceCanAccessPeer(&ok, a, b));
            if (!ok)
                return gfail(g, TXS_ERR_CUDA, "[site] group: device " + std::to_string(a) + " cannot access device " +
                                                  std::to_string(b) + "'s memory (use TXS_XCHG_NCCL)");
            G_CUDA(g, "peer access", cudaSetDevice(a));
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_gfail(g, "peer access", e);
            cudaGetLastError();
        }
    g->peers_enabled = true;
    return TXS_OK;
}

txs_status ensure_comms(txs_group* g) {
    if (!g->comms.empty()) return TXS_OK;
    if (!distinct_devices(g)) return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[site] group: NCCL needs one rank per device");
    if (!nccl().ok) return gfail(g, TXS_ERR_CUDA, "[site] group: libnccl.so.2 not loadable");
    g->comms.assign((size_t)g->n, nullptr);
    const ncclResult_t r = nccl().CommInitAll(g->comms.data(), g->n, g->dev.data());
    if (r != ncclSuccess) {
        g->comms.clear();
        return gfail(g, TXS_ERR_CUDA, std::string("[site] group: ncclCommInitAll: ") + nccl().GetErrorString(r));
    }
    return TXS_OK;
}

txs_status alloc_round_buffers(txs_group* g, int64_t pw) {
    if (g->pw == pw && !g->d_key.empty()) return TXS_OK;
    free_round_buffers(g);
    const size_t n = (size_t)g->n;
    g->d_key.assign(n, nullptr); g->d_pay.assign(n, nullptr); g->d_gather.assign(n, nullptr);
    for (int b = 0; b < 2; ++b) { g->d_mail[b].assign(n, nullptr); g->d_peers[b].assign(n, nullptr); }
    for (int k = 0; k < g->n; ++k) {
        G_CUDA(g, "buffers", cudaSetDevice(g->dev[(size_t)k]));
        G_CUDA(g, "buffers", cudaMalloc(&g->d_key[(size_t)k], 8));
        G_CUDA(g, "buffers", cudaMalloc(&g->d_pay[(size_t)k], 8 * (size_t)pw));
        G_CUDA(g, "buffers", cudaMemset(g->d_pay[(size_t)k], 0, 8 * (size_t)pw));
        for (int b = 0; b < 2; ++b) {
            G_CUDA(g, "buffers", cudaMalloc(&g->d_mail[b][(size_t)k], 8 * (size_t)(pw + 1)));
            G_CUDA(g, "buffers", cudaMemset(g->d_mail[b][(size_t)k], 0, 8 * (size_t)(pw + 1)));
        }
        if (g->exchange == TXS_XCHG_NCCL)
            G_CUDA(g, "buffers", cudaMalloc(&g->d_gather[(size_t)k], 8 * (size_t)(pw + 1) * n));
    }
    for (int k = 0; k < g->n; ++k) {   // every rank's table of the N mailboxes (peer pointers)
        G_CUDA(g, "buffers", cudaSetDevice(g->dev[(size_t)k]));
        for (int b = 0; b < 2; ++b) {
            G_CUDA(g, "buffers", cudaMalloc(&g->d_peers[b][(size_t)k], sizeof(uint64_t*) * n));
            G_CUDA(g, "buffers", cudaMemcpy(g->d_peers[b][(size_t)k], g->d_mail[b].data(), sizeof(uint64_t*) * n,
                                            cudaMemcpyHostToDevice));
        }
    }
    g->pw = pw;
    return TXS_OK;
}

// one SITE round of every rank, stream-ordered (eager or under capture)
txs_status enqueue_round(txs_group* g, int parity, int64_t total) {
    const int n = g->n;
    txs_status st = TXS_OK;
    for (int k = 0; k < n; ++k) {
        txs_ctx* c = g->ctx[(size_t)k];
        uint64_t* mail = g->exchange == TXS_XCHG_NCCL ? g->d_mail[0][(size_t)k] : g->d_mail[parity][(size_t)k];
        if ((st = txs_site_shard_best_dev(c, g->d_key[(size_t)k])) != TXS_OK ||
            (st = txs_site_shard_export_keyed_dev(c, g->d_key[(size_t)k], mail)) != TXS_OK)
            return rank_fail(g, k, st);
        if (g->exchange == TXS_XCHG_P2P) G_CUDA(g, "round", cudaEventRecord(g->ev_mail[parity][(size_t)k], c->stream));
    }
    if (g->exchange == TXS_XCHG_NCCL) {
        NcclApi& N = nccl();
        ncclResult_t r = N.GroupStart();
        for (int k = 0; k < n && r == ncclSuccess; ++k) {
            cudaSetDevice(g->dev[(size_t)k]);
            r = N.AllGather(g->d_mail[0][(size_t)k], g->d_gather[(size_t)k], (size_t)(g->pw + 1), ncclUint64,
                            g->comms[(size_t)k], g->ctx[(size_t)k]->stream);
        }
        const ncclResult_t r2 = N.GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return gfail(g, TXS_ERR_CUDA, std::string("[site] group: ncclAllGather: ") +
                                              N.GetErrorString(r != ncclSuccess ? r : r2));
    }
    for (int k = 0; k < n; ++k) {
        txs_ctx* c = g->ctx[(size_t)k];
        G_CUDA(g, "round", cudaSetDevice(g->dev[(size_t)k]));
        if (g->exchange == TXS_XCHG_P2P) {
            for (int j = 0; j < n; ++j)
                if (j != k) G_CUDA(g, "round", cudaStreamWaitEvent(c->stream, g->ev_mail[parity][(size_t)j], 0));
            st = txs::shard_site_select_peers(c, g->d_peers[parity][(size_t)k], n, g->d_key[(size_t)k],
                                              g->d_pay[(size_t)k]);
        } else {
            st = txs_site_shard_select_dev(c, g->d_gather[(size_t)k], n, g->d_key[(size_t)k], g->d_pay[(size_t)k]);
        }
        if (st != TXS_OK) return rank_fail(g, k, st);
        if ((st = txs_site_shard_apply_dev(c, g->d_key[(size_t)k], g->d_pay[(size_t)k], total)) != TXS_OK)
            return rank_fail(g, k, st);
    }
    return TXS_OK;
}

// kGraphRounds rounds of every rank as one multi-device graph on rank 0's stream
txs_status capture_rounds(txs_group* g, int first_parity, int64_t total) {
    if (g->graph) { cudaGraphExecDestroy(g->graph); g->graph = nullptr; }
    cudaStream_t s0 = g->ctx[0]->stream;
    G_CUDA(g, "capture", cudaSetDevice(g->dev[0]));
    G_CUDA(g, "capture", cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
    txs_status st = TXS_OK;
    cudaError_t e = cudaEventRecord(g->ev_fork, s0);
    for (int k = 1; k < g->n && e == cudaSuccess; ++k) {
        cudaSetDevice(g->dev[(size_t)k]);
        e = cudaStreamWaitEvent(g->ctx[(size_t)k]->stream, g->ev_fork, 0);
    }
    for (int t = 0; t < kGraphRounds && e == cudaSuccess && st == TXS_OK; ++t)
        st = enqueue_round(g, (first_parity + t) & 1, total);
    for (int k = 1; k < g->n && e == cudaSuccess && st == TXS_OK; ++k) {
        cudaSetDevice(g->dev[(size_t)k]);
        e = cudaEventRecord(g->ev_join[(size_t)k], g->ctx[(size_t)k]->stream);
        cudaSetDevice(g->dev[0]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, g->ev_join[(size_t)k], 0);
    }
    cudaSetDevice(g->dev[0]);
    cudaGraph_t graph = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(s0, &graph);
    if (st != TXS_OK) { if (graph) cudaGraphDestroy(graph); return st; }
    if (e != cudaSuccess) { if (graph) cudaGraphDestroy(graph); return cuda_gfail(g, "capture", e); }
    if (e2 != cudaSuccess) return cuda_gfail(g, "capture", e2);
    e = cudaGraphInstantiate(&g->graph, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) { g->graph = nullptr; return cuda_gfail(g, "graph instantiate", e); }
    return TXS_OK;
}

txs_status device_rounds(txs_group* g, int64_t total, std::vector<txs_step>& steps, int32_t* stop, double* ms) {
    txs_status st = ensure_events(g);
    if (st != TXS_OK) return st;
    if (g->exchange == TXS_XCHG_P2P && (st = enable_peers(g)) != TXS_OK) return st;
    if (g->exchange == TXS_XCHG_NCCL && (st = ensure_comms(g)) != TXS_OK) return st;
    const int64_t pw = txs_site_shard_payload_words(g->ctx[0]);
    if ((st = alloc_round_buffers(g, pw)) != TXS_OK) return st;
    for (int k = 0; k < g->n; ++k) G_CUDA(g, "sync", (cudaSetDevice(g->dev[(size_t)k]), cudaStreamSynchronize(g->ctx[(size_t)k]->stream)));
    cudaSetDevice(g->dev[0]);
    G_CUDA(g, "timing", cudaEventRecord(g->ev_t0, g->ctx[0]->stream));
    // one eager round (sizes every rank's device step log), then graph replays
    if ((st = enqueue_round(g, 0, total)) != TXS_OK) return st;
    for (int k = 1; k < g->n; ++k) {   // rank 0's stream joins the others: a graph launched on it follows
        G_CUDA(g, "join", cudaSetDevice(g->dev[(size_t)k]));
        G_CUDA(g, "join", cudaEventRecord(g->ev_join[(size_t)k], g->ctx[(size_t)k]->stream));
        G_CUDA(g, "join", cudaSetDevice(g->dev[0]));
        G_CUDA(g, "join", cudaStreamWaitEvent(g->ctx[0]->stream, g->ev_join[(size_t)k], 0));
    }
    if ((st = capture_rounds(g, 1, total)) != TXS_OK) return st;
    int64_t ns = 0;
    int32_t sr = -1;
    for (int64_t done = 1;; done += kGraphRounds) {
        cudaSetDevice(g->dev[0]);
        if ((st = txs_site_shard_result(g->ctx[0], nullptr, 0, &ns, &sr)) != TXS_OK) return rank_fail(g, 0, st);
        if (sr >= 0 || done > total + 1 + kGraphRounds) break;
        G_CUDA(g, "replay", cudaGraphLaunch(g->graph, g->ctx[0]->stream));   // ends joined on rank 0's stream
    }
    if (sr < 0) return gfail(g, TXS_ERR_STATE, "[site] group: SITE rounds did not stop");
    cudaSetDevice(g->dev[0]);
    G_CUDA(g, "timing", cudaEventRecord(g->ev_t1, g->ctx[0]->stream));
    G_CUDA(g, "timing", cudaEventSynchronize(g->ev_t1));
    float f = 0.f;
    G_CUDA(g, "timing", cudaEventElapsedTime(&f, g->ev_t0, g->ev_t1));
    *ms = f;
    steps.resize((size_t)std::max<int64_t>(ns, 0));
    if ((st = txs_site_shard_result(g->ctx[0], steps.data(), ns, &ns, &sr)) != TXS_OK) return rank_fail(g, 0, st);
    *stop = sr;
    for (int k = 1; k < g->n; ++k) {   // every rank must have taken the same decisions
        int64_t nk = 0;
        int32_t sk = -1;
        if ((st = txs_site_shard_result(g->ctx[(size_t)k], nullptr, 0, &nk, &sk)) != TXS_OK) return rank_fail(g, k, st);
        if (nk != ns || sk != sr) return gfail(g, TXS_ERR_STATE, "[site] group: ranks disagree on the SITE sequence");
    }
    return TXS_OK;
}

// TXS_XCHG_REPLICATE: every band's viewsheds packed as records on its own
// device, copied once into rank 0's HBM (peer copies over NVLink), then rank 0
// runs the single-GPU SITE loop on the gathered set (txs_site_gathered)
txs_status replicated_site(txs_group* g, const txs_params& p, int64_t total, std::vector<txs_step>& steps,
                           int32_t* stop, double* ms) {
    const int n = g->n;
    const int64_t rw = txs_viewshed_record_words(p.roi);
    std::vector<int64_t> cnt((size_t)n, 0);
    int64_t nmax = 1;
    for (int k = 0; k < n; ++k) {
        cnt[(size_t)k] = g->ctx[(size_t)k]->vs_n;
        nmax = std::max(nmax, cnt[(size_t)k]);
    }
    G_CUDA(g, "gather", cudaSetDevice(g->dev[0]));
    uint64_t* d_all = nullptr;
    G_CUDA(g, "gather", cudaMalloc(&d_all, sizeof(uint64_t) * (size_t)(n * nmax * rw)));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, g->ctx[0]->stream);
    txs_status st = for_ranks(g, [&](int k) {   // pack on each device, then one peer copy into rank 0
        txs_ctx* c = g->ctx[(size_t)k];
        uint64_t* dst = d_all + (size_t)k * nmax * rw;
        if (g->dev[(size_t)k] == g->dev[0]) return txs_viewsheds_pack(c, nmax, dst, nullptr);
        cudaSetDevice(g->dev[(size_t)k]);
        uint64_t* tmp = nullptr;
        if (cudaMalloc(&tmp, sizeof(uint64_t) * (size_t)(nmax * rw)) != cudaSuccess) return TXS_ERR_OUT_OF_MEMORY;
        txs_status s2 = txs_viewsheds_pack(c, nmax, tmp, nullptr);
        if (s2 == TXS_OK &&
            (cudaMemcpyPeerAsync(dst, g->dev[0], tmp, g->dev[(size_t)k], sizeof(uint64_t) * (size_t)(nmax * rw), c->stream) !=
                 cudaSuccess ||
             cudaStreamSynchronize(c->stream) != cudaSuccess))
            s2 = TXS_ERR_CUDA;
        cudaFree(tmp);
        return s2;
    });
    if (st == TXS_OK) {
        for (int k = 0; k < n; ++k) cudaStreamSynchronize(g->ctx[(size_t)k]->stream);
        cudaSetDevice(g->dev[0]);
        cudaEventRecord(e1, g->ctx[0]->stream);
        cudaEventSynchronize(e1);
        float f = 0.f;
        cudaEventElapsedTime(&f, e0, e1);
        steps.resize((size_t)total + 1);
        int64_t ns = 0;
        const txs_stats before = g->ctx[0]->stats;
        st = txs_site_gathered(g->ctx[0], &p, n * nmax, total, d_all, steps.data(), (int64_t)steps.size(), &ns, stop);
        if (st != TXS_OK) st = rank_fail(g, 0, st);
        steps.resize((size_t)std::max<int64_t>(0, ns));
        *ms = f + (g->ctx[0]->stats.ms_site - before.ms_site);
    }
    cudaSetDevice(g->dev[0]);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_all);
    if (st == TXS_OK) g->replicated = true;
    return st;
}

// host-staged rounds (TXS_XCHG_HOST): shard.py's host loop, stop rules D9
txs_status host_rounds(txs_group* g, const txs_params& p, int64_t total, std::vector<txs_step>& steps,
                       int32_t* stop) {
    const int64_t stride = txs::max_window_words(g->roi);
    std::vector<uint64_t> words((size_t)stride);
    const double area = (double)g->nrows * (double)g->ncols;
    int64_t covered = 0;
    txs_status st = TXS_OK;
    for (;;) {
        if ((int64_t)steps.size() >= total) { *stop = TXS_STOP_EXHAUSTED; return TXS_OK; }
        uint64_t key = 0;
        for (int k = 0; k < g->n; ++k) {
            uint64_t kk = 0;
            if ((st = g->ops.site_shard_best(g->ctx[(size_t)k], &kk)) != TXS_OK) return rank_fail(g, k, st);
            key = std::max(key, kk);
        }
        const int64_t gain = (int64_t)(key >> 32);
        if (gain <= 0) { *stop = TXS_STOP_ZERO_GAIN; return TXS_OK; }
        const int64_t gid = (int64_t)(0xffffffffull - (key & 0xffffffffull));
        int32_t owned = 0, row = 0, col = 0;
        txs_window win{};
        for (int k = 0; k < g->n && !owned; ++k)
            if ((st = g->ops.site_shard_export(g->ctx[(size_t)k], gid, &owned, &row, &col, &win, words.data(), stride)) != TXS_OK)
                return rank_fail(g, k, st);
        if (!owned) return gfail(g, TXS_ERR_STATE, "[site] group: no rank owns the winning candidate");
        for (int k = 0; k < g->n; ++k)
            if ((st = g->ops.site_shard_apply(g->ctx[(size_t)k], row, col, &win, words.data())) != TXS_OK)
                return rank_fail(g, k, st);
        covered += gain;
        const double cov = (double)covered / area;
        steps.push_back(txs_step{gid, row, col, gain, cov});
        if (cov >= p.target_coverage) { *stop = TXS_STOP_TARGET_REACHED; return TXS_OK; }
        if (p.max_selected > 0 && (int64_t)steps.size() >= p.max_selected) { *stop = TXS_STOP_MAX_SELECTED; return TXS_OK; }
    }
}

}  // namespace

extern "C" {

const txs_engine_ops* txs_default_ops(void) { return &kDefaultOps; }

txs_status txs_plan_bands(int64_t nrows, int64_t block, int32_t world, int64_t* out) {
    if (nrows < 1 || block < 1 || world < 1 || !out) return TXS_ERR_INVALID_ARGUMENT;
    const int64_t nb = (nrows + block - 1) / block;
    if (world > nb) return TXS_ERR_INVALID_ARGUMENT;   // a rank would own no block row
    const int64_t base = nb / world, extra = nb % world;
    int64_t b = 0;
    for (int32_t k = 0; k < world; ++k) {
        const int64_t cnt = base + (k < extra ? 1 : 0);
        out[2 * k] = std::min(nrows, b * block);
        out[2 * k + 1] = std::min(nrows, (b + cnt) * block);
        b += cnt;
    }
    return TXS_OK;
}

txs_status txs_group_create_with_ops(int ngpus, const int* devices, const txs_engine_ops* ops, txs_group** out) {
    if (!out || ngpus < 1 || ngpus > 64 || !ops) return TXS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    txs_group* g = new txs_group();
    g->ops = *ops;
    g->native = ops == &kDefaultOps;
    g->exchange = g->native ? TXS_XCHG_REPLICATE : TXS_XCHG_HOST;
    g->n = ngpus;
    for (int k = 0; k < ngpus; ++k) g->dev.push_back(devices ? devices[k] : k);
    for (int k = 0; k < ngpus; ++k) {
        txs_ctx* c = nullptr;
        const txs_status st = g->ops.create(g->dev[(size_t)k], &c);
        if (st != TXS_OK) {
            txs_group_destroy(g);
            return st;
        }
        g->ctx.push_back(c);
    }
    *out = g;
    return TXS_OK;
}

txs_status txs_group_create(int ngpus, const int* devices, txs_group** out) {
    return txs_group_create_with_ops(ngpus, devices, &kDefaultOps, out);
}

void txs_group_destroy(txs_group* g) {
    if (!g) return;
    if (g->native) {
        free_round_buffers(g);
        destroy_events(g);
        for (ncclComm_t c : g->comms) if (c) nccl().CommDestroy(c);
    }
    for (txs_ctx* c : g->ctx) if (c) g->ops.destroy(c);
    delete g;
}

const char* txs_group_last_error(const txs_group* g) { return g ? g->err.c_str() : "null group"; }
int32_t txs_group_size(const txs_group* g) { return g ? g->n : 0; }
txs_ctx* txs_group_context(txs_group* g, int32_t rank) {
    return (g && rank >= 0 && rank < g->n) ? g->ctx[(size_t)rank] : nullptr;
}

txs_status txs_group_set_exchange(txs_group* g, int32_t x) {
    if (!g) return TXS_ERR_INVALID_ARGUMENT;
    if (x != TXS_XCHG_P2P && x != TXS_XCHG_NCCL && x != TXS_XCHG_HOST && x != TXS_XCHG_REPLICATE)
        return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[site] group: unknown exchange");
    if (!g->native && x != TXS_XCHG_HOST)
        return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[site] group: substituted ops support the host exchange only");
    if (x == TXS_XCHG_NCCL && !distinct_devices(g))
        return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[site] group: NCCL needs one rank per device");
    if (x != g->exchange && g->native) free_round_buffers(g);
    g->exchange = x;
    return TXS_OK;
}

txs_status txs_group_set_grid(txs_group* g, int64_t nrows, int64_t ncols, const txs_params* p) {
    if (!g || !p) return TXS_ERR_INVALID_ARGUMENT;
    if (p->roi < 1) return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[vix] roi must be >= 1");
    const int64_t block = p->block_width > 0 ? p->block_width : (p->roi + 2) / 3;
    std::vector<int64_t> b((size_t)(2 * g->n));
    if (txs_plan_bands(nrows, block, g->n, b.data()) != TXS_OK)
        return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[read] group: more ranks than FINDMAX block rows (" +
                                                      std::to_string((nrows + block - 1) / std::max<int64_t>(1, block)) + ")");
    g->nrows = nrows; g->ncols = ncols; g->block = block; g->roi = p->roi;
    g->r0.assign((size_t)g->n, 0); g->r1.assign((size_t)g->n, 0);
    for (int k = 0; k < g->n; ++k) { g->r0[(size_t)k] = b[(size_t)(2 * k)]; g->r1[(size_t)k] = b[(size_t)(2 * k + 1)]; }
    g->observers = -1;
    return for_ranks(g, [&](int k) {
        return g->ops.set_shard(g->ctx[(size_t)k], nrows, ncols, g->r0[(size_t)k], g->r1[(size_t)k], p->roi + 1);
    });
}

txs_status txs_group_band(const txs_group* g, int32_t rank, int64_t* rb, int64_t* re) {
    if (!g || rank < 0 || rank >= g->n || !rb || !re || g->r0.empty()) return TXS_ERR_INVALID_ARGUMENT;
    *rb = g->r0[(size_t)rank];
    *re = g->r1[(size_t)rank];
    return TXS_OK;
}

txs_status txs_group_set_terrain(txs_group* g, const int16_t* z) {
    if (!g || !z) return TXS_ERR_INVALID_ARGUMENT;
    if (g->r0.empty()) return gfail(g, TXS_ERR_STATE, "[read] group: call txs_group_set_grid first");
    g->observers = -1;
    return for_ranks(g, [&](int k) {
        int64_t h0 = 0, hr = 0, b0 = 0, b1 = 0;
        txs_status st = g->ops.shard_info(g->ctx[(size_t)k], &h0, &hr, &b0, &b1);
        if (st != TXS_OK) return st;
        return g->ops.set_terrain(g->ctx[(size_t)k], z + h0 * g->ncols, hr, g->ncols);
    });
}

txs_status txs_group_generate_fractal(txs_group* g, double roughness, uint64_t seed, int32_t zmin, int32_t zmax) {
    if (!g) return TXS_ERR_INVALID_ARGUMENT;
    if (g->r0.empty()) return gfail(g, TXS_ERR_STATE, "[read] group: call txs_group_set_grid first");
    g->observers = -1;
    return for_ranks(g, [&](int k) {
        return g->ops.generate_fractal(g->ctx[(size_t)k], g->nrows, g->ncols, roughness, seed, zmin, zmax);
    });
}

txs_status txs_group_fill_rows(txs_group* g, int64_t rb, int64_t re, int16_t v) {
    if (!g) return TXS_ERR_INVALID_ARGUMENT;
    if (g->r0.empty()) return gfail(g, TXS_ERR_STATE, "[read] group: call txs_group_set_grid first");
    return for_ranks(g, [&](int k) { return g->ops.fill_rows(g->ctx[(size_t)k], rb, re, v); });
}

txs_status txs_group_random_observers(txs_group* g, int64_t n, uint64_t seed) {
    if (!g || n < 0) return TXS_ERR_INVALID_ARGUMENT;
    if (g->r0.empty()) return gfail(g, TXS_ERR_STATE, "[read] group: call txs_group_set_grid first");
    const txs_status st = for_ranks(g, [&](int k) { return g->ops.random_observers(g->ctx[(size_t)k], n, seed); });
    g->observers = st == TXS_OK ? n : -1;
    return st;
}

txs_status txs_group_run_pipeline(txs_group* g, const txs_params* p, txs_step* steps, int64_t cap, int64_t* nsteps,
                                  int32_t* stop_reason, double* stage_ms) {
    if (!g || !p) return TXS_ERR_INVALID_ARGUMENT;
    if (g->r0.empty()) return gfail(g, TXS_ERR_STATE, "[read] group: call txs_group_set_grid first");
    if (p->roi != g->roi) return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[viewshed] group: roi differs from txs_group_set_grid's");
    if (!(p->target_coverage > 0.0) || p->target_coverage > 1.0)
        return gfail(g, TXS_ERR_INVALID_ARGUMENT, "[site] target_coverage must be in (0,1]");
    const size_t n = (size_t)g->n;
    std::vector<txs_stats> before(n), after(n);
    std::vector<int64_t> count(n, 0);
    txs_status st = for_ranks(g, [&](int k) { return g->ops.get_stats(g->ctx[(size_t)k], &before[(size_t)k]); });
    if (st != TXS_OK) return st;
    // ---- VIX + FINDMAX per band (or the band's random observers) ----
    st = for_ranks(g, [&](int k) {
        txs_ctx* c = g->ctx[(size_t)k];
        if (g->observers >= 0) return g->ops.get_candidates(c, nullptr, 0, &count[(size_t)k]);
        txs_status s = g->ops.estimate_vix(c, p, nullptr);
        return s != TXS_OK ? s : g->ops.find_candidates(c, p, &count[(size_t)k], nullptr, 0);
    });
    if (st != TXS_OK) return st;
    int64_t total = 0;
    if (g->observers >= 0) {
        total = g->observers;   // ids are the global draw indices
    } else {
        for (int k = 0; k < g->n; ++k) {   // global id = prefix of the band counts + local index
            if ((st = g->ops.set_candidate_base(g->ctx[(size_t)k], total)) != TXS_OK) return rank_fail(g, k, st);
            total += count[(size_t)k];
        }
    }
    // ---- VIEWSHED per band ----
    const bool repl = g->exchange == TXS_XCHG_REPLICATE;
    g->replicated = false;
    st = for_ranks(g, [&](int k) {
        txs_status s = g->ops.compute_viewsheds(g->ctx[(size_t)k], p);
        return (s != TXS_OK || repl) ? s : g->ops.site_shard_begin(g->ctx[(size_t)k], p);
    });
    if (st != TXS_OK) return st;
    // ---- SITE rounds ----
    std::vector<txs_step> v;
    int32_t sr = TXS_STOP_EXHAUSTED;
    double site_ms = 0.0;
    if (repl) {
        st = replicated_site(g, *p, total, v, &sr, &site_ms);
    } else if (g->exchange == TXS_XCHG_HOST) {
        const auto t0 = std::chrono::steady_clock::now();
        st = host_rounds(g, *p, total, v, &sr);
        site_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } else {
        st = device_rounds(g, total, v, &sr, &site_ms);
    }
    if (st != TXS_OK) return st;
    if (nsteps) *nsteps = (int64_t)v.size();
    if (stop_reason) *stop_reason = sr;
    if (steps) std::copy(v.begin(), v.begin() + std::min<int64_t>(cap, (int64_t)v.size()), steps);
    if (stage_ms) {
        st = for_ranks(g, [&](int k) { return g->ops.get_stats(g->ctx[(size_t)k], &after[(size_t)k]); });
        if (st != TXS_OK) return st;
        stage_ms[0] = stage_ms[1] = stage_ms[2] = 0.0;
        for (size_t k = 0; k < n; ++k) {   // the stage ends when its slowest band does
            stage_ms[0] = std::max(stage_ms[0], after[k].ms_vix - before[k].ms_vix);
            stage_ms[1] = std::max(stage_ms[1], after[k].ms_findmax - before[k].ms_findmax);
            stage_ms[2] = std::max(stage_ms[2], after[k].ms_viewshed - before[k].ms_viewshed);
        }
        stage_ms[3] = site_ms;
    }
    return TXS_OK;
}

txs_status txs_group_get_cumulative(txs_group* g, uint64_t* dense_out) {
    if (!g || !dense_out) return TXS_ERR_INVALID_ARGUMENT;
    if (g->r0.empty()) return gfail(g, TXS_ERR_STATE, "[site] group: no grid");
    std::memset(dense_out, 0, sizeof(uint64_t) * (size_t)((g->nrows * g->ncols + 63) / 64));
    if (g->replicated) {   // rank 0 holds the whole grid's cum
        const txs_status st = txs_get_cumulative(g->ctx[0], dense_out);
        return st == TXS_OK ? st : rank_fail(g, 0, st);
    }
    return for_ranks(g, [&](int k) {
        return g->ops.get_cumulative_rows(g->ctx[(size_t)k], g->r0[(size_t)k], g->r1[(size_t)k], dense_out);
    });
}

}  // extern "C"
