// swamp_gpu.cu — host side of the C-ABI (include/swamp_gpu.h): owns device
// memory, sequences the sm_100a kernels of hwfv1_kernels.cuh, captures one
// adaptive step (K1 -> K2 -> K3 -> K5) as a CUDA graph and replays it.
//
// Boundary: replaces the reference's engine operations initialise /
// step_adaptive / step_uniform / run for the adaptive
// time-step loop. No CPU fallback: every compute path is a CUDA kernel; a
// missing device is an error.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "hwfv1_kernels.cuh"
#include "swamp_gpu.h"

using hwfv1::Ctl;
using hwfv1::kThreads;
using hwfv1::Params;

namespace {

constexpr int kGraphSteps = 8;

struct Mem {
    void* p = nullptr;
    ~Mem() {
        if (p) cudaFree(p);
    }
};

// Process-wide cache of device blocks and pinned control mirrors: an engine's
// buffers go back here when it is destroyed and the next engine of the same
// shape reuses them. cudaMalloc / cudaFree of the ~400 MB an L = 11 engine
// holds cost 3-50 ms each time (measured on B200), which would otherwise land
// in every initialise. Capped at kCacheCap bytes per process;
// swamp_gpu_trim_cache() releases it. (Never destroyed: freeing at process
// exit would race the CUDA runtime's own teardown.)
constexpr size_t kCacheCap = size_t(16) << 30;
struct BlockCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void*> dev;  // (device, bytes) -> block
    std::vector<void*> pinned;                          // sizeof(Ctl) host blocks
    size_t bytes = 0;
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache;
    return *c;
}
cudaError_t cached_malloc(int device, void** p, size_t bytes) {
    BlockCache& c = block_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.dev.find({device, bytes});
        if (it != c.dev.end()) {
            *p = it->second;
            c.dev.erase(it);
            c.bytes -= bytes;
            return cudaSuccess;
        }
    }
    return cudaMalloc(p, bytes);
}
void cached_free(int device, void* p, size_t bytes) {
    BlockCache& c = block_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.bytes + bytes <= kCacheCap) {
            c.dev.insert({{device, bytes}, p});
            c.bytes += bytes;
            return;
        }
    }
    cudaFree(p);
}
// step reports in flight in swamp_gpu_advance_reports (a power of two)
constexpr int kRepRing = 16;
cudaError_t cached_pinned_ctl(Ctl** p) {
    BlockCache& c = block_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        if (!c.pinned.empty()) {
            *p = static_cast<Ctl*>(c.pinned.back());
            c.pinned.pop_back();
            return cudaSuccess;
        }
    }
    return cudaMallocHost(reinterpret_cast<void**>(p), (1 + kRepRing) * sizeof(Ctl));  // (the control mirror + the report ring)
}
void cached_free_pinned_ctl(Ctl* p) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.pinned.push_back(p);
}

}  // namespace

struct swamp_gpu {
    int device = 0;
    bool uniform = false;
    bool profiling = false;
    cudaStream_t stream = nullptr;
    Params P{};
    Ctl* ctl = nullptr;      // device
    Ctl* ctl_host = nullptr; // pinned mirror
    std::vector<std::pair<void*, size_t>> allocs;  // device blocks (returned to the block cache)
    cudaGraphExec_t graph1 = nullptr, graphS = nullptr, graphT = nullptr, graphR = nullptr;
    // advance_reports: 8-step / 1-step graphs whose finalize writes each
    // step's report into the pinned ring (ctl_host + 1 .. + kRepRing)
    cudaGraphExec_t graphQ = nullptr, graphQ1 = nullptr;
    Ctl* ring_dev = nullptr;
    int fv1_grid = 0;
    int64_t launches_per_step = 0;  // kernel nodes of the one-step graph
    bool mirror_current = false;    // ctl_host holds the state after the last completed step
    // k_fv1 STAGE (SWAMP_FV1_STAGE): 2: own cell and subtree activity loaded
    // an iteration ahead (FV1 69 -> 66 us); 3: also the neighbours'
    // parent-level flags (65 us; default below L = 11); 5: 3 + the last
    // grid-stride windows handed out dynamically (64 us; default from L = 11);
    // 0: L2 prefetch only
    int fv1_stage = 5;
    bool k2_split = false;   // K2's top encode as its own launch (k_band_top), one partition, split K3
    size_t smem_k2top = 0;
    int num_sms = 0;
    size_t smem_k1 = 0, smem_k1s = 0, smem_k2 = 0, smem_k3 = 0;
    // K3 split into a top launch (alone on its SM) + a subtree launch (one partition)
    void (*k3top)(Params, Ctl*) = nullptr;
    void (*k3tiles)(Params, Ctl*) = nullptr;
    size_t smem_k3top = 0, smem_k3tiles = 0;
    // fused K2 + K3 (k_23, one cooperative grid): K2 not launched
    void (*k23)(Params, Ctl*) = nullptr;
    size_t smem_k23 = 0;
    // tile kernels, specialised for K = 6 (every L >= 6) or generic
    void (*k1)(Params, Ctl*) = nullptr;
    void (*k2)(Params, Ctl*, int, int) = nullptr;
    void (*k3)(Params, Ctl*, int, unsigned long long) = nullptr;
    void (*k3x)(Params, Ctl*, int, unsigned long long) = nullptr;
    unsigned long long export_epoch = 1ull << 62;  // K3 export launches (hot-path epochs are 2 step + 2)
    cudaEvent_t ev[6] = {};
    std::string err;
    int64_t n_cells = 0;
    // partitioned group: the shell owns one sub-engine per
    // partition (each with full-size arrays on its device); empty otherwise
    std::vector<swamp_gpu*> parts;
    // one partition of a multi-process (rank) engine: peer mappings opened
    // from other processes' CUDA IPC handles, closed on destruction
    int rank_world = 0;
    std::vector<void*> ipc_opened;
    bool serial = false;  // group on one device: all partitions on parts[0]'s stream
    bool concurrent = false;  // (serial group) phases run as concurrent per-partition branches
    cudaEvent_t ev_fork = nullptr;
    cudaEvent_t ev_join[hwfv1::kMaxParts] = {};
    void* scratch = nullptr;  // device scratch of export_finest (3 x 4^L doubles), lazily allocated
    double x0 = 0.0, y0 = 0.0;  // lower-left corner of the domain (gauge sampling)
    size_t scratch_bytes = 0;

    ~swamp_gpu() {
        // no kernel of any partition may still read a block (its own, or a
        // peer's through the peer tables / IPC mappings) once it is returned
        // to the cache or unmapped: drain every device involved first
        for (swamp_gpu* q : parts) {
            cudaSetDevice(q->device);
            cudaDeviceSynchronize();
        }
        for (swamp_gpu* q : parts) {
            cudaSetDevice(q->device);
            delete q;
        }
        if (!ipc_opened.empty() || !allocs.empty() || scratch) {
            cudaSetDevice(device);
            cudaDeviceSynchronize();
        }
        for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
        if (scratch) cached_free(device, scratch, scratch_bytes);
        if (graph1) cudaGraphExecDestroy(graph1);
        if (graphS) cudaGraphExecDestroy(graphS);
        if (ev_fork) cudaEventDestroy(ev_fork);
        for (cudaEvent_t e : ev_join)
            if (e) cudaEventDestroy(e);
        if (graphT) cudaGraphExecDestroy(graphT);
        if (graphR) cudaGraphExecDestroy(graphR);
        if (graphQ) cudaGraphExecDestroy(graphQ);
        if (graphQ1) cudaGraphExecDestroy(graphQ1);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (!allocs.empty() || scratch) cudaSetDevice(device);
        for (auto& a : allocs) cached_free(device, a.first, a.second);
        if (ctl_host) cached_free_pinned_ctl(ctl_host);
        if (stream) cudaStreamDestroy(stream);
    }
};

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            if (g) g->err = std::string(#call) + ": " + cudaGetErrorString(e_);       \
            return SWAMP_E_CUDA;                                                      \
        }                                                                             \
    } while (0)

namespace {

template <class T>
int dalloc(swamp_gpu* g, T** out, size_t bytes) {
    void* p = nullptr;
    bytes = std::max<size_t>(bytes, 16);
    cudaError_t e = cached_malloc(g->device, &p, bytes);
    if (e != cudaSuccess) {
        g->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
        return SWAMP_E_NOMEM;
    }
    g->allocs.push_back({p, bytes});
    *out = static_cast<T*>(p);
    return SWAMP_OK;
}

int validate(const swamp_config* c) {
    if (!c) return SWAMP_E_ARG;
    if (c->L < 1 || c->L > 13) return SWAMP_E_ARG;
    if (!(c->epsilon >= 0.0) || !(c->width > 0.0) || !(c->cfl > 0.0 && c->cfl <= 1.0)) return SWAMP_E_ARG;
    if (!(c->h_dry > 0.0) || !(c->g > 0.0) || !(c->manning >= 0.0) || !(c->dt_fallback > 0.0)) return SWAMP_E_ARG;
    for (int k = 0; k < 4; ++k)
        if (c->bc[k] < 0 || c->bc[k] > 2) return SWAMP_E_ARG;
    if (c->band_mode < 0 || c->band_mode > 2) return SWAMP_E_ARG;
    if (c->inflow_n < 0 || (c->inflow_n > 0 && (!c->inflow_t || !c->inflow_v))) return SWAMP_E_ARG;
    if (c->inflow_mode != SWAMP_INFLOW_DEPTH && c->inflow_mode != SWAMP_INFLOW_ETA) return SWAMP_E_ARG;
    for (int k = 0; k < 4; ++k)  // an inflow edge without a series would silently become a dry ghost
        if (c->bc[k] == SWAMP_BC_INFLOW && c->inflow_n == 0) return SWAMP_E_ARG;
    if (c->n_outputs < 0 || (c->n_outputs > 0 && !c->output_times)) return SWAMP_E_ARG;
    return SWAMP_OK;
}

// launch with programmatic stream serialisation (PDL, see pdl_wait/pdl_trigger)
template <class... KArgs, class... Args>
void launch_pdl_t(void (*kernel)(KArgs...), int grid, int threads, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}
// PDL + cooperative (every CTA of the grid resident at once, or the launch fails)
template <class... KArgs, class... Args>
void launch_pdl_coop(void (*kernel)(KArgs...), int grid, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, size_t smem, cudaStream_t s, Args... args) {
    launch_pdl_t(kernel, grid, kThreads, smem, s, args...);
}
// plain stream-ordered launch (the kernels' griddepcontrol.wait is then a no-op)
template <class... KArgs, class... Args>
void launch_plain_t(void (*kernel)(KArgs...), int grid, int threads, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.numAttrs = 0;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

void launch_step_kernels(swamp_gpu* g, bool timed) {
    Params& P = g->P;
    cudaStream_t s = g->stream;
    // event record NODES inside a captured graph need the External flag
    auto mark = [&](int k) {
        if (timed) cudaEventRecordWithFlags(g->ev[k], s, cudaEventRecordExternal);
    };
    mark(0);
    if (g->uniform) {
        if (P.has_ina)
            launch_pdl(hwfv1::k_fv1<true, false, true>, g->fv1_grid, 0, s, P, g->ctl);
        else
            launch_pdl(hwfv1::k_fv1<true>, g->fv1_grid, 0, s, P, g->ctl);
        for (int k = 1; k < 5; ++k) mark(k);
        return;
    }
    launch_pdl(g->k1, P.n_tiles + (P.rep_ring ? 1 : 0), g->smem_k1s, s, P, g->ctl);  // (+1: the ring's report CTA)
    if (P.top_mode == 2) launch_pdl(hwfv1::k_encode_top<false>, 1, g->smem_k1, s, P, g->ctl);
    mark(1);
    if (g->k23) {  // fused K2 + K3
        mark(2);
        launch_pdl_coop(g->k23, P.n_tiles + 1, g->smem_k23, s, P, g->ctl);
        mark(3);
    } else {
    if (g->k2_split) {  // the top encode on its own SM, then the subtree grid
        launch_pdl(hwfv1::k_band_top, 1, g->smem_k2top, s, P, g->ctl);
        launch_pdl(g->k2, P.n_tiles, g->smem_k2, s, P, g->ctl, 0, 2);
    } else {
        const int do_top = P.top_mode == 1 ? 1 : 0;
        launch_pdl(g->k2, P.n_tiles + do_top, g->smem_k2, s, P, g->ctl, 0, do_top);
    }
    mark(2);
    if (g->k3top) {
        launch_pdl_t(g->k3top, 1, hwfv1::kTopThreads, g->smem_k3top, s, P, g->ctl);
        launch_pdl(g->k3tiles, P.n_tiles, g->smem_k3tiles, s, P, g->ctl);
    } else {
        launch_pdl(g->k3, P.n_tiles + 1, g->smem_k3, s, P, g->ctl, 0, 0ull);
    }
    mark(3);
    }
    const size_t fsm = P.tiles ? hwfv1::kTileSlab : 0;  // the tile phase's row slabs
    if (P.has_ina)  // D16 variant
        launch_pdl(hwfv1::k_fv1<false, false, true>, g->fv1_grid, 0, s, P, g->ctl);
    else if (g->fv1_stage == 2)
        launch_pdl(hwfv1::k_fv1<false, false, false, 2>, g->fv1_grid, fsm, s, P, g->ctl);
    else if (g->fv1_stage == 3)
        launch_pdl(hwfv1::k_fv1<false, false, false, 3>, g->fv1_grid, fsm, s, P, g->ctl);
    else if (g->fv1_stage == 5)
        launch_pdl(hwfv1::k_fv1<false, false, false, 5>, g->fv1_grid, fsm, s, P, g->ctl);
    else
        launch_pdl(hwfv1::k_fv1<false>, g->fv1_grid, fsm, s, P, g->ctl);
    mark(4);
}

// graph1: one step; graphS: kGraphSteps steps; graphT: one step with event
// record nodes between the kernels (per-stage device times, StepReport)
// `which`: 0 = graph1, 1 = graphS, 2 = graphT (the profiling graph is built
// on first use)
// kernel nodes of a captured one-step graph (swamp_gpu_counters [5])
int64_t kernel_nodes(cudaGraph_t graph) {
    size_t n = 0;
    if (cudaGraphGetNodes(graph, nullptr, &n) != cudaSuccess || n == 0) return 0;
    std::vector<cudaGraphNode_t> nodes(n);
    if (cudaGraphGetNodes(graph, nodes.data(), &n) != cudaSuccess) return 0;
    int64_t k = 0;
    for (cudaGraphNode_t v : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(v, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
}

// which: 0 graph1 (one step), 1 graphS (kGraphSteps), 2 graphT (one step,
// event nodes), 3 graphR (one step whose FV1 also writes the host mirror:
// step_adaptive's report; the mirror write costs ~2 us, so only graphR has it)
int build_graph(swamp_gpu* g, int which) {
    {
        const int steps = (which == 1 || which == 4) ? kGraphSteps : 1;
        Ctl* const mirror = g->P.ctl_mirror;
        if (which != 3) g->P.ctl_mirror = nullptr;
        if (which >= 4) g->P.rep_ring = g->ring_dev;
        cudaGraph_t graph;
        cudaError_t e = cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            for (int k = 0; k < steps; ++k) launch_step_kernels(g, which == 2);
            e = cudaStreamEndCapture(g->stream, &graph);
        }
        g->P.ctl_mirror = mirror;
        g->P.rep_ring = nullptr;
        CK(e);
        if (which == 0) g->launches_per_step = kernel_nodes(graph);
        cudaGraphExec_t exec;
        CK(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        (which == 0 ? g->graph1 : which == 1 ? g->graphS : which == 2 ? g->graphT : which == 3 ? g->graphR
                                                                          : which == 4 ? g->graphQ : g->graphQ1) = exec;
    }
    return SWAMP_OK;
}
int build_graphs(swamp_gpu* g) {  // graph1, the 8-step graph and graphR now (timed loops replay them), graphT on demand
    int st = build_graph(g, 0);
    if (!st) st = build_graph(g, 1);
    if (!st && g->P.ctl_mirror) st = build_graph(g, 3);
    // advance_reports' graphs: built here (overlapped with the initial tree)
    // for the large engines; small ones build them on first use (each costs
    // ~0.1 ms of host time, a visible share of a short run's creation)
    const bool q = g->ring_dev && !g->uniform && g->P.n_tiles >= 1024;
    if (!st && q) st = build_graph(g, 4);
    if (!st && q) st = build_graph(g, 5);
    return st;
}
// single engines: the 8-step graph / the profiling graph on demand
int ensure_graph(swamp_gpu* g, int which) {
    cudaGraphExec_t e = which == 1 ? g->graphS : which == 2 ? g->graphT : which == 4 ? g->graphQ
                        : which == 5 ? g->graphQ1 : g->graph1;
    if (e || !g->parts.empty() || g->rank_world > 0) return SWAMP_OK;
    return build_graph(g, which);
}

int fetch_ctl(swamp_gpu* g) {
    CK(cudaMemcpyAsync(g->ctl_host, g->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    g->mirror_current = true;
    if (g->ctl_host->err_code != 0) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "device error %d at z=%u quantity=%d stage=%d", g->ctl_host->err_code,
                      g->ctl_host->err_z, g->ctl_host->err_q, g->ctl_host->err_stage);
        g->err = buf;
        return g->ctl_host->err_code;
    }
    return SWAMP_OK;
}

// stage times of the last completed step from the device timeline (globaltimer)
void fill_stage_times(const swamp_gpu* g, const Ctl& c, swamp_step_report* r) {
    if (c.step <= 0) return;
    const auto& tl = c.tl[(c.step - 1) & 1];
    // kernel k: from its first CTA's start to its last CTA's end
    auto start = [&](int k) { return tl[k][0] ? ~tl[k][0] : 0ull; };
    auto span = [&](int ka, int kb) -> double {
        const unsigned long long s0 = start(ka), s1 = tl[kb][2];
        return (s0 == 0 || s1 == 0 || s1 < s0) ? 0.0 : 1e-6 * static_cast<double>(s1 - s0);
    };
    if (g->uniform) {
        r->ms_fv1 = span(3, 3);
        r->ms_total = r->ms_fv1;
        return;
    }
    r->ms_encode_flag = span(0, 0);
    r->ms_band_closure = span(1, 1);
    r->ms_decode_traverse = span(2, 2);
    r->ms_neighbours = 0.0;
    r->ms_fv1 = span(3, 3);
    r->ms_total = span(0, 3);
}

// a report from control-block words c (the host copy, the mirror or a ring slot)
void fill_report_from(const swamp_gpu* g, const Ctl& c, swamp_step_report* r) {
    if (!r) return;
    std::memset(r, 0, sizeof(*r));
    fill_stage_times(g, c, r);
    r->step = c.step;
    r->t = c.t;
    r->dt = c.dt;
    r->dt_used = c.dt_used;
    r->n_leaves = g->uniform ? (int64_t(1) << (2 * g->P.L)) : c.n_leaves_used;
    r->n_leaves_next = g->uniform ? r->n_leaves : c.n_leaves;
    r->n_near_threshold = g->uniform ? 0 : static_cast<int64_t>(c.near_last);
}
void fill_report(const swamp_gpu* g, swamp_step_report* r) { fill_report_from(g, *g->ctl_host, r); }

// a partitioned group's report: partition 0's, with the near-threshold
// count summed over the partitions (each counts its own subtrees)
void fill_group_report(const swamp_gpu* grp, swamp_step_report* r) {
    if (!r) return;
    fill_report(grp->parts[0], r);
    int64_t nn = 0;
    for (const swamp_gpu* q : grp->parts) nn += static_cast<int64_t>(q->ctl_host->near_last);
    r->n_near_threshold = nn;
}

// allocate + upload + import one (sub-)engine: everything before the
// initialise pipeline. Partition `part` of `G` owns level-R subtrees
// [part, part+1) * 4^R / G.
// SWAMP_TRACE=1: wall time of the creation phases on stderr (diagnostics)
struct Trace {
    bool on = false;
    std::chrono::steady_clock::time_point t0;
    Trace() {
        const char* e = std::getenv("SWAMP_TRACE");
        on = e && e[0] == '1';
        t0 = std::chrono::steady_clock::now();
    }
    void operator()(const char* what) const {
        if (on)
            std::fprintf(stderr, "[swamp] %-28s %8.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

int setup_part(swamp_gpu* g, const swamp_config* cfg, const double* h, const double* qx, const double* qy,
               const double* z, int device, int G, int part) {
    int st = SWAMP_OK;
    const Trace tr;
    auto fail = [&](int code) { return code; };
    g->device = device;
    if (cudaSetDevice(device) != cudaSuccess) return fail(SWAMP_E_CUDA);
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(SWAMP_E_CUDA);
    for (auto& e : g->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return fail(SWAMP_E_CUDA);
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);
    tr("stream + events");

    Params& P = g->P;
    const int L = cfg->L;
    P.L = L;
    P.K = std::min(L, 6);
    P.R = L - P.K;
    P.n_tiles = 1 << (2 * P.R);
    if (G < 1 || G > hwfv1::kMaxParts || P.n_tiles % G != 0) return SWAMP_E_ARG;
    P.G = G;
    P.part = part;
    P.tiles_per_part = static_cast<uint32_t>(P.n_tiles / G);
    P.tile_lo = static_cast<uint32_t>(part) * P.tiles_per_part;
    P.tile_hi = P.tile_lo + P.tiles_per_part;
    for (int k = 0; k <= hwfv1::kMaxParts; ++k)
        P.pbound[k] = static_cast<uint32_t>(std::min(k, G)) * P.tiles_per_part;
    P.pb_align = (P.tiles_per_part % 16 == 0) ? 16u : (P.tiles_per_part % 4 == 0) ? 4u : 1u;
    P.band_mode = cfg->band_mode;
    for (int k = 0; k < 4; ++k) P.bc[k] = cfg->bc[k];
    P.inflow_mode = cfg->inflow_mode;
    P.inflow_n = cfg->inflow_n;
    P.n_out = cfg->n_outputs;
    P.W = cfg->width;
    g->x0 = cfg->x0;
    g->y0 = cfg->y0;
    P.cfl = cfg->cfl;
    P.t_end = cfg->t_end;
    P.dt_fallback = cfg->dt_fallback;
    P.phys.g = cfg->g;
    P.phys.half_g = 0.5 * cfg->g;
    P.phys.hdry = cfg->h_dry;
    P.phys.nM = cfg->manning;
    P.phys.g_nM2 = cfg->g * (cfg->manning * cfg->manning);
    for (int n = 0; n <= L; ++n) {
        P.dx[n] = std::ldexp(cfg->width, -n);
        P.inv_dx[n] = 1.0 / P.dx[n];
    }
    // level layout: each level's slice rounded up to 8 cells (256 B)
    unsigned long long off = 0, foff = 0;
    for (int n = 0; n <= L; ++n) {
        P.base[n] = off;
        off += ((1ull << (2 * n)) + 7ull) & ~7ull;
    }
    for (int n = 0; n < L; ++n) {
        P.fbase[n] = foff;
        foff += ((1ull << (2 * n)) + 15ull) & ~15ull;
    }
    // the kernels use closed forms of the level tables (hwfv1_kernels.cuh)
    for (int n = 0; n < L; ++n)
        if (P.fbase[n] != hwfv1::slo(n)) return fail(SWAMP_E_ARG);
    for (int n = 0; n <= L; ++n) {
        if (P.base[n] != hwfv1::cbase(n)) return fail(SWAMP_E_ARG);
        long long b0, bn;
        std::memcpy(&b0, &P.inv_dx[0], 8);
        std::memcpy(&bn, &P.inv_dx[n], 8);
        if (bn != b0 + (static_cast<long long>(n) << 52)) return fail(SWAMP_E_ARG);
    }
    g->n_cells = static_cast<int64_t>(off);
    const size_t nf = static_cast<size_t>(1) << (2 * L);
    if ((st = dalloc(g, &P.cells[0], off * sizeof(double4)))) return fail(st);
    if ((st = dalloc(g, &P.cells[1], off * sizeof(double4)))) return fail(st);
    if ((st = dalloc(g, &P.sig[0], foff))) return fail(st);
    if ((st = dalloc(g, &P.sig[1], foff))) return fail(st);
    if ((st = dalloc(g, &P.pre, foff))) return fail(st);
    if ((st = dalloc(g, &P.dem, foff))) return fail(st);
    if ((st = dalloc(g, &P.leaves, nf * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.leaves_x, nf * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.tile_cnt, 2 * P.n_tiles * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.tile_off, 3 * P.n_tiles * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.tile_lvl, P.n_tiles * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.wet[0], P.n_tiles))) return fail(st);
    if ((st = dalloc(g, &P.wet[1], P.n_tiles))) return fail(st);
    if ((st = dalloc(g, &P.tact, P.n_tiles))) return fail(st);
    if ((st = dalloc(g, &P.qwet[0], 4 * P.n_tiles))) return fail(st);
    if ((st = dalloc(g, &P.qwet[1], 4 * P.n_tiles))) return fail(st);
    if ((st = dalloc(g, &P.stile, P.n_tiles * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.tchg, P.n_tiles))) return fail(st);
    {
        double* smx = nullptr;
        if ((st = dalloc(g, &smx, 8 * sizeof(double)))) return fail(st);
        P.smx = smx;
    }
    if ((st = dalloc(g, &P.qstate, P.n_tiles))) return fail(st);
    if ((st = dalloc(g, &P.qnk1, 2 * P.n_tiles * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.qnfv, P.n_tiles * sizeof(uint32_t)))) return fail(st);
    cudaMemsetAsync(P.tchg, 1, P.n_tiles, g->stream);
    cudaMemsetAsync(P.qstate, 0, P.n_tiles, g->stream);
    cudaMemsetAsync(P.qnk1, 0, 2 * P.n_tiles * sizeof(uint32_t), g->stream);
    cudaMemsetAsync(P.qnfv, 0, P.n_tiles * sizeof(uint32_t), g->stream);

    P.pdem[0] = P.dem;
    P.pwet[0][0] = P.wet[0];
    P.pwet[0][1] = P.wet[1];
    P.has_ina = cfg->inactive ? 1 : 0;
    if (P.has_ina && (st = dalloc(g, &P.ina, hwfv1::slo(L + 1) + 16))) return fail(st);
    // every subtree counts as wet until FV1 has run once
    cudaMemsetAsync(P.wet[0], 1, P.n_tiles, g->stream);
    cudaMemsetAsync(P.wet[1], 1, P.n_tiles, g->stream);
    cudaMemsetAsync(P.qwet[0], 1, 4 * P.n_tiles, g->stream);
    cudaMemsetAsync(P.qwet[1], 1, 4 * P.n_tiles, g->stream);
    cudaMemsetAsync(P.tact, 1, P.n_tiles, g->stream);
    if ((st = dalloc(g, &P.tile_src, P.n_tiles * sizeof(uint32_t)))) return fail(st);
    if ((st = dalloc(g, &P.k3_rec, P.n_tiles * 4 * sizeof(unsigned long long)))) return fail(st);
    // K3's per-subtree records carry an epoch tag (2 step + 2, so initialise's
    // K3 polls for tag 2): a block reused from the cache may hold records of
    // an engine that stopped after its first step, which that poll would
    // accept — clear them before anything runs
    cudaMemsetAsync(P.k3_rec, 0, P.n_tiles * 4 * sizeof(unsigned long long), g->stream);
    if ((st = dalloc(g, &g->ctl, sizeof(Ctl)))) return fail(st);
    // peer tables: self only (a partitioned group fills in every partition)
    for (int b = 0; b < 2; ++b) {
        P.pcells[0][b] = P.cells[b];
        P.psig[0][b] = P.sig[b];
    }
    P.ppre[0] = P.pre;
    P.ptile_cnt[0] = P.tile_cnt;
    P.pctl[0] = g->ctl;
    tr("device allocations");
    if (cached_pinned_ctl(&g->ctl_host) != cudaSuccess) return fail(SWAMP_E_NOMEM);
    P.ctl_mirror = nullptr;
    if (G == 1) {  // FV1's finalizing CTA writes each step's control block into the pinned mirror
        void* dm = nullptr;
        const char* em = std::getenv("SWAMP_MIRROR");
        if (!(em && em[0] == '0') && cudaHostGetDevicePointer(&dm, g->ctl_host, 0) == cudaSuccess) {
            P.ctl_mirror = static_cast<Ctl*>(dm);
            g->ring_dev = P.ctl_mirror + 1;
        }
    }
    P.rep_ring = nullptr;  // (set only while advance_reports' graphs are captured)
    P.rep_ring_mask = kRepRing - 1;
    tr("pinned control block");
    double *d_it = nullptr, *d_iv = nullptr, *d_out = nullptr;
    if ((st = dalloc(g, &d_it, sizeof(double) * std::max(1, cfg->inflow_n)))) return fail(st);
    if ((st = dalloc(g, &d_iv, sizeof(double) * std::max(1, cfg->inflow_n)))) return fail(st);
    if ((st = dalloc(g, &d_out, sizeof(double) * std::max(1, cfg->n_outputs)))) return fail(st);
    cudaStream_t s = g->stream;
    if (cfg->inflow_n > 0) {
        cudaMemcpyAsync(d_it, cfg->inflow_t, sizeof(double) * cfg->inflow_n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_iv, cfg->inflow_v, sizeof(double) * cfg->inflow_n, cudaMemcpyHostToDevice, s);
    }
    if (cfg->n_outputs > 0)
        cudaMemcpyAsync(d_out, cfg->output_times, sizeof(double) * cfg->n_outputs, cudaMemcpyHostToDevice, s);
    P.inflow_t = d_it;
    P.inflow_v = d_iv;
    P.out_times = d_out;

    // control block
    Ctl c0{};
    std::memcpy(g->ctl_host, &c0, sizeof(Ctl));
    if (cudaMemcpyAsync(g->ctl, g->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, s) != cudaSuccess)
        return fail(SWAMP_E_CUDA);

    // upload + import (the staging buffer is released right after)
    {
        // DMA the host rasters (full speed from page-locked memory) into the
        // second cell buffer, free until initialise copies buffer 0 into it
        const double* src[4] = {h, qx, qy, z};
        double* stage = reinterpret_cast<double*>(P.cells[1]);
        static_assert(sizeof(double4) == 4 * sizeof(double), "layout");
        const double* dsrc[4];
        for (int q = 0; q < 4; ++q) {
            cudaMemcpyAsync(stage + q * nf, src[q], nf * sizeof(double), cudaMemcpyHostToDevice, s);
            dsrc[q] = stage + q * nf;
        }
        uint8_t* mask = nullptr;
        if (P.has_ina) {
            mask = reinterpret_cast<uint8_t*>(stage + 4 * nf);  // (cells[1] holds 4 nf doubles + 1/8 more)
            cudaMemcpyAsync(mask, cfg->inactive, nf, cudaMemcpyHostToDevice, s);
        }
        const int grid = std::max(1, std::min<int>(g->num_sms * 8, static_cast<int>((nf + kThreads - 1) / kThreads)));
        hwfv1::k_import<<<grid, kThreads, 0, s>>>(P, g->ctl, dsrc[0], dsrc[1], dsrc[2], dsrc[3], mask, 0);
        for (int n = L - 1; P.has_ina && n >= 0; --n) {
            const int gl = std::max(1, std::min<int>(g->num_sms * 4, static_cast<int>(((1u << (2 * n)) + kThreads - 1) / kThreads)));
            hwfv1::k_ina_level<<<gl, kThreads, 0, s>>>(P, n);
        }
        // s_max table on the device: nothing below waits for the upload (the
        // host goes on with the tables, kernel attributes and, in create,
        // the step graphs while the rasters stream in; a non-finite input is
        // reported by the error word at the end of creation)
        hwfv1::k_smax_table<<<1, 32, 0, s>>>(g->ctl, const_cast<double*>(P.smx));
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            g->err = cudaGetErrorString(e);
            return fail(SWAMP_E_CUDA);
        }
    }
    tr("upload + import (enqueued)");
    // significance table (D7, D8; hwfv1::sig_class): SPEC's
    // max|d| / s_max >= eps 2^(n-L) on s = p 2^(L-n) coefficients is
    // fl(max|D| / s_max) >= e_n = eps 2^(2n-2L+2) on physical details D (the
    // same rounding: the two differ by exact powers of two); near-threshold
    // band tol = 1e-12 e_n; screening window e_n (1 -/+ 1e-11)
    for (int n = 0; n < L; ++n) {
        const double e = std::ldexp(cfg->epsilon, 2 * n - 2 * L + 2);
        P.tau[n] = e;
        P.lvl[n][0] = e * (1.0 - 1e-11);
        P.lvl[n][1] = e * (1.0 + 1e-11);
        P.lvl[n][2] = 1e-12 * e;
        P.lvl[n][3] = e;
    }

    // shared memory per kernel (hwfv1_kernels.cuh layouts)
    {
        const int Ki = P.K;
        const size_t K = P.K, R = P.R, nt = P.n_tiles;
        const size_t ncell = ((size_t(1) << (2 * K)) - 1) / 3;      // subtree cells, levels R..L-1
        const size_t fb = P.fbase[R];                                // top flag bytes (levels < R)
        const size_t ltop = ((size_t(1) << (2 * R)) - 1) / 3;        // top cells (levels < R)
        const size_t sl = hwfv1::slo(Ki);
        if (Ki == 6) {
            g->k1 = hwfv1::k_encode_step<6>;
            g->k2 = hwfv1::k_band<6>;
            g->k3 = hwfv1::k_traverse<false, 6>;
            g->k3x = hwfv1::k_traverse<true, 6>;
        } else {
            g->k1 = hwfv1::k_encode_step<0>;
            g->k2 = hwfv1::k_band<0>;
            g->k3 = hwfv1::k_traverse<false, 0>;
            g->k3x = hwfv1::k_traverse<true, 0>;
        }
        g->smem_k1 = ncell * (sizeof(double4) + 1);                  // k_encode<true> / k_encode_top
        g->smem_k1s = 32 * (((size_t(1) << (2 * (K - 1))) - 1) / 3) + 4 * sl;  // values, 2 flag copies, DEM, new pre
        P.top_mode = (R == 0) ? 0 : (R <= 6 ? 1 : 2);
        const size_t k2_tile = 3 * sl;  // pre flags, band / final flags, previous flags (quiet skip)
        const char* etb = std::getenv("SWAMP_TOP_BAND");
        P.top_band = (P.top_mode == 1 && G == 1 && !(etb && etb[0] == '0')) ? 1 : 0;
        const size_t k2_top = P.top_mode == 1 ? 32 * ltop + 3 * fb : 0;
        g->smem_k2 = std::max(k2_tile, k2_top);
        const size_t ftop = (fb + nt + 15) & ~size_t(15);
        const size_t k3_top_smem = 2 * ftop + 2 * ((nt + 15) & ~size_t(15)) + 2 * fb + (nt <= 1024 ? 8 * nt : 0);
        g->smem_k3 = std::max(2 * sl + 4 * ncell, k3_top_smem);  // subtree CTA, top CTA
        // split K3 (SWAMP_K3_SPLIT=0: one launch with the top as block 0)
        const char* eks = std::getenv("SWAMP_K3_SPLIT");
        if (G == 1 && P.top_mode == 1 && !(eks && eks[0] == '0')) {
            g->k3top = (Ki == 6) ? hwfv1::k_traverse_top<6> : hwfv1::k_traverse_top<0>;
            g->k3tiles = (Ki == 6) ? hwfv1::k_traverse_tiles<6> : hwfv1::k_traverse_tiles<0>;
            g->smem_k3tiles = 2 * sl + 4 * ncell;
            int smem_optin = 0;
            cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
            g->smem_k3top = std::max(k3_top_smem, static_cast<size_t>(smem_optin) - 8 * 1024);
            // K2's top encode on its own SM (SWAMP_K2_SPLIT=0: block 0 of K2)
            const char* eks2 = std::getenv("SWAMP_K2_SPLIT");
            g->k2_split = P.top_band && !(eks2 && eks2[0] == '0');
            g->smem_k2top = std::max(k2_top, static_cast<size_t>(smem_optin) - 8 * 1024);
            // FV1 tile path (active fully refined subtrees as 64 x 64 blocks,
            // every face once): one partition, K = 6, no inactive cells, the
            // split K3 (its top lists the tiles); SWAMP_FV1_TILES=0 disables
            // Below L = 11 a strip's serial rows are the step's critical path
            // (few jobs per CTA): humps L9 39 -> 31 us/step without the tile
            // phase, Monai L10 74 -> 71; SWAMP_FV1_TILES=0 / 1 forces it
            const char* et = std::getenv("SWAMP_FV1_TILES");
            const bool tl = et ? et[0] != '0' : P.n_tiles >= 1024;
            P.tiles = (Ki == 6 && !P.has_ina && tl) ? 1 : 0;
            // quiet split of the leaf lists (SWAMP_QSPLIT=0 disables)
            const char* eq = std::getenv("SWAMP_QSPLIT");
            P.qsplit = (!P.has_ina && !(eq && eq[0] == '0')) ? 1 : 0;
            // quadrant wet marks for the activity test (SWAMP_QACT=0 disables)
            const char* eqa = std::getenv("SWAMP_QACT");
            P.qact = (P.qsplit && !(eqa && eqa[0] == '0')) ? 1 : 0;
            // stable-quiet skip (needs the quiet split and K = 6: one K1 CTA
            // per subtree). Config 5: 117 -> 97 us/step; below L = 11 its
            // bookkeeping in K2 / K3 costs ~1 us more than it saves.
            // SWAMP_QSKIP=0 / 1 forces it off / on
            const char* eqs = std::getenv("SWAMP_QSKIP");
            const bool qk = eqs ? eqs[0] != '0' : P.n_tiles >= 1024;
            P.qskip = (P.qsplit && Ki == 6 && qk) ? 1 : 0;
            // fused K2 + K3 (k_23, one cooperative grid): needs top_band (K2's
            // extra-CTA work moves into the top CTA) and every CTA resident at
            // once (the top waits for all subtree CTAs, they wait for its
            // records; the cooperative launch guarantees the residency).
            // Measured -3 us per step at L = 8..10; +2 to +3 us at L = 11 (one
            // 1024-subtree wave behind a 256-thread top), so on below 1024
            // subtrees. SWAMP_K23=0 / 1 forces it off / on
            const char* e23 = std::getenv("SWAMP_K23");
            const bool k23 = e23 ? e23[0] == '1' : P.n_tiles < 1024;
            if (P.top_band && k23) {
                void (*f23)(Params, Ctl*) = (Ki == 6) ? hwfv1::k_23<6> : hwfv1::k_23<0>;
                // (the top's own layout, not the split top's whole-SM request)
                const hwfv1::K3TopLayout ly = hwfv1::k3_top_layout(R, static_cast<uint32_t>(nt));
                const size_t top23 = ly.sqw + 4 * ((nt + 15) & ~size_t(15)) + 64;
                const size_t sm23 = std::max(sl + g->smem_k3tiles, top23);
                int occ = 0;
                if (sm23 >= 32 * 1024)
                    cudaFuncSetAttribute(reinterpret_cast<const void*>(f23),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm23));
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f23, kThreads, sm23);
                if (static_cast<long long>(occ) * g->num_sms >= P.n_tiles + 1) {
                    g->k23 = f23;
                    g->smem_k23 = sm23;
                    P.qact = 0;  // (the fused top does not refine by quadrants)
                }
            }
        }
        struct {
            const void* f;
            size_t bytes;
        } attrs[] = {{reinterpret_cast<const void*>(g->k1), g->smem_k1s},
                     {reinterpret_cast<const void*>(hwfv1::k_encode<true>), g->smem_k1},
                     {reinterpret_cast<const void*>(hwfv1::k_encode_top<true>), g->smem_k1},
                     {reinterpret_cast<const void*>(hwfv1::k_encode_top<false>), g->smem_k1},
                     {reinterpret_cast<const void*>(g->k2), g->smem_k2},
                     {reinterpret_cast<const void*>(g->k3), g->smem_k3},
                     {reinterpret_cast<const void*>(g->k3x), g->smem_k3},
                     {reinterpret_cast<const void*>(g->k3top), g->smem_k3top},
                     {reinterpret_cast<const void*>(hwfv1::k_band_top), g->k2_split ? g->smem_k2top : 0},
                     {reinterpret_cast<const void*>(g->k3tiles), g->smem_k3tiles},
                     {reinterpret_cast<const void*>(g->k23), g->smem_k23},
                     {reinterpret_cast<const void*>(hwfv1::k_fv1<false>), hwfv1::kTileSlab},
                     {reinterpret_cast<const void*>(hwfv1::k_fv1<false, false, false, 2>), hwfv1::kTileSlab},
                     {reinterpret_cast<const void*>(hwfv1::k_fv1<false, false, false, 3>), hwfv1::kTileSlab},
                     {reinterpret_cast<const void*>(hwfv1::k_fv1<false, false, false, 5>), hwfv1::kTileSlab}};
        for (auto& a : attrs)
            if (a.f && a.bytes >= 32 * 1024 &&
                cudaFuncSetAttribute(a.f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(a.bytes)) !=
                    cudaSuccess)
                return fail(SWAMP_E_CUDA);
    }
    {
        // tail balancing pays when the leaf list spans many grid-stride
        // windows (L = 11: ~22); below that its bookkeeping costs ~5 %
        g->fv1_stage = (L >= 11) ? 5 : 3;
        if (const char* e = std::getenv("SWAMP_FV1_STAGE")) g->fv1_stage = std::atoi(e);
        // tail balancing: the last 6/16 of FV1's grid-stride windows go to
        // whichever warps are free (8 of 22 windows at L = 11: FV1 66.3 ->
        // 64.3 us; 2-6 windows less, 10-24 windows less to slower)
        const char* etw = std::getenv("SWAMP_FV1_TAIL16");
        P.fv1_tail16 = etw ? static_cast<uint32_t>(std::min(16, std::max(0, std::atoi(etw)))) : 6u;
        // several lanes per leaf when the list fits the grid that way (STAGE 3)
        const char* efp = std::getenv("SWAMP_FV1_FP_CAP16");
        P.fv1_fp_cap16 = efp ? static_cast<uint32_t>(std::min(256, std::max(0, std::atoi(efp)))) : 16u;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hwfv1::k_fv1<false, false, false, 5>, kThreads, 0);
        g->fv1_grid = std::max(1, occ) * g->num_sms;
        if (const char* eg = std::getenv("SWAMP_FV1_GRID_PCT"))  // (A/B: grid as a percentage of one wave)
            g->fv1_grid = std::max(g->num_sms, g->fv1_grid * std::max(10, std::atoi(eg)) / 100);
    }
    g->n_cells = static_cast<int64_t>(off);
    tr("kernel attributes");
    return SWAMP_OK;
}

int create_impl(const swamp_config* cfg, const double* h, const double* qx, const double* qy, const double* z,
                int device, bool uniform, swamp_gpu** out) {
    if (!out || !h || !qx || !qy || !z) return SWAMP_E_ARG;
    *out = nullptr;
    int st = validate(cfg);
    if (st) return st;
    auto* g = new swamp_gpu();
    g->uniform = uniform;
    auto fail = [&](int code) {
        delete g;
        return code;
    };
    const Trace tr;
    if ((st = setup_part(g, cfg, h, qx, qy, z, device, 1, 0))) return fail(st);
    tr("setup");
    Params& P = g->P;
    cudaStream_t s = g->stream;
    const unsigned long long off = static_cast<unsigned long long>(g->n_cells);
    const unsigned long long foff = P.fbase[P.L - 1] + (((1ull << (2 * (P.L - 1))) + 15ull) & ~15ull);

    if (uniform) {
        // full tree, no MRA: every detail cell significant
        cudaMemsetAsync(P.sig[0], 1, foff, s);
        cudaMemsetAsync(P.sig[1], 1, foff, s);
        cudaMemsetAsync(P.pre, 1, foff, s);
        // leaf list = every finest cell in Morton order (for exports)
        g->k2<<<P.n_tiles, kThreads, g->smem_k2, s>>>(P, g->ctl, 1, 0);
        g->k3<<<P.n_tiles + 1, kThreads, g->smem_k3, s>>>(P, g->ctl, 1, 0ull);
        cudaMemcpyAsync(P.cells[1], P.cells[0], off * sizeof(double4), cudaMemcpyDeviceToDevice, s);
        hwfv1::k_cfl_init<<<g->fv1_grid, kThreads, 0, s>>>(P, g->ctl, 1);
    } else {
        // initialise: previous tree := everything, full
        // encode + DEM mask, band + closure, traversal; no decode at t = 0
        cudaMemsetAsync(P.sig[0], 1, foff, s);
        hwfv1::k_encode<true><<<P.n_tiles, kThreads, g->smem_k1, s>>>(P, g->ctl);
        if (P.has_ina) hwfv1::k_ina_mix<<<std::max(1, g->num_sms * 4), kThreads, 0, s>>>(P);
        g->k2<<<P.n_tiles, kThreads, g->smem_k2, s>>>(P, g->ctl, 1, 0);
        g->k3<<<P.n_tiles + 1, kThreads, g->smem_k3, s>>>(P, g->ctl, 1, 0ull);
        // both buffers hold the full hierarchy; the current tree becomes "previous"
        cudaMemcpyAsync(P.cells[1], P.cells[0], off * sizeof(double4), cudaMemcpyDeviceToDevice, s);
        hwfv1::k_set_parity<<<1, 32, 0, s>>>(g->ctl, 1);
        hwfv1::k_near_l1<<<g->num_sms * 4, kThreads, 0, s>>>(P, g->ctl);
        hwfv1::k_cfl_init<<<g->fv1_grid, kThreads, 0, s>>>(P, g->ctl, 0);
    }
    // the step graphs are captured and instantiated on the host while the
    // device builds the initial tree (capture records new work only; the
    // launches queued above run on)
    if ((st = build_graphs(g))) return fail(st);
    tr("graphs (host)");
    {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            g->err = cudaGetErrorString(e);
            return fail(SWAMP_E_CUDA);
        }
        if (cudaGetLastError() != cudaSuccess) return fail(SWAMP_E_CUDA);
    }
    tr("initial tree");
    {
        // export_finest's device scratch, taken now (from the block cache when
        // an engine of this shape existed before) so an export never pays a
        // cudaMalloc (3-90 ms for 100 MB at L = 11, measured)
        const size_t nf = static_cast<size_t>(1) << (2 * P.L);
        if (cached_malloc(g->device, &g->scratch, 3 * nf * sizeof(double)) != cudaSuccess) {
            g->scratch = nullptr;
            return fail(SWAMP_E_NOMEM);
        }
        g->scratch_bytes = 3 * nf * sizeof(double);
    }
    if ((st = fetch_ctl(g))) return fail(st);
    cudaMemsetAsync(g->ctl->tl, 0, sizeof(g->ctl->tl), s);
    cudaMemsetAsync(&g->ctl->k3_ready, 0, sizeof(g->ctl->k3_ready), s);  // hot-path epochs restart at step 0
    cudaMemsetAsync(P.k3_rec, 0, P.n_tiles * 4 * sizeof(unsigned long long), s);  // (and the per-subtree records)
    tr("ready");
    *out = g;
    return SWAMP_OK;
}


// ============================================================ partitioned
// Morton-subtree partitions. Partition `part` of G owns level-R
// subtrees [part, part + 1) * 4^R / G; peers' arrays are read in place through
// the peer tables (NVLink peer access between devices, CUDA IPC mappings
// between processes). Every partition runs the same kernel sequence on its
// own stream with a device-side barrier (k_part_barrier) between phases, so a
// partition's step is a fixed sequence that is captured as a CUDA graph and
// replayed independently of the others: a group of partitions in one process
// (swamp_gpu_create_partitioned) and one partition per process
// (swamp_gpu_rank_*) share this code.
void part_barrier(swamp_gpu* q, cudaStream_t s) { launch_pdl_t(hwfv1::k_part_barrier, 1, 32, 0, s, q->P, q->ctl); }

// phase k of a partitioned step on stream s (k = 0..5: K1, top encode, K2,
// K3, FV1, finalize); false when the phase does not apply
// (every phase kernel and the barrier start with griddepcontrol.wait, so the
// phases are chained with programmatic dependent launch: each launch overlaps
// the tail of the kernel before it)
bool part_step_phase(swamp_gpu* q, int k, cudaStream_t s, bool pdl = true) {
    const Params& P = q->P;
    // (PDL between phases on one stream; the concurrent same-device group
    // joins the partitions' streams between phases, so plain launches there)
    auto launch = [&](auto kernel, int grid, int threads, size_t smem, auto... args) {
        if (pdl) launch_pdl_t(kernel, grid, threads, smem, s, args...);
        else launch_plain_t(kernel, grid, threads, smem, s, args...);
    };
    switch (k) {
        case 0:
            launch(q->k1, static_cast<int>(P.tiles_per_part), kThreads, q->smem_k1s, P, q->ctl);
            return true;
        case 1:
            if (P.top_mode != 2) return false;
            launch(hwfv1::k_encode_top<false>, 1, kThreads, q->smem_k1, P, q->ctl);
            return true;
        case 2: {
            const int do_top = P.top_mode == 1 ? 1 : 0;
            launch(q->k2, static_cast<int>(P.tiles_per_part) + do_top, kThreads, q->smem_k2, P, q->ctl, 0, do_top);
            return true;
        }
        case 3: launch(q->k3, static_cast<int>(P.tiles_per_part) + 1, kThreads, q->smem_k3, P, q->ctl, 0, 0ull); return true;
        case 4:
            if (P.has_ina) launch(hwfv1::k_fv1<false, true, true>, q->fv1_grid, kThreads, 0, P, q->ctl);
            else if (q->fv1_stage == 5)  // tail balancing (flags come from the peer tables: no STAGE 3 preloads)
                launch(hwfv1::k_fv1<false, true, false, 5>, q->fv1_grid, kThreads, 0, P, q->ctl);
            else if (q->fv1_stage >= 2)  // own cells loaded an iteration ahead
                launch(hwfv1::k_fv1<false, true, false, 2>, q->fv1_grid, kThreads, 0, P, q->ctl);
            else
                launch(hwfv1::k_fv1<false, true>, q->fv1_grid, kThreads, 0, P, q->ctl);
            return true;
        default: launch(hwfv1::k_finalize, 1, 32, 0, P, q->ctl, 1); return true;
    }
}
constexpr int kStepPhases = 6;

// phase k of initialise on stream s (k = 0..5)
bool part_init_phase(swamp_gpu* q, int k, cudaStream_t s) {
    const Params& P = q->P;
    switch (k) {
        case 0: {
            const size_t foff = P.fbase[P.L - 1] + (((size_t(1) << (2 * (P.L - 1))) + 15) & ~size_t(15));
            cudaMemsetAsync(P.sig[0], 1, foff, s);
            hwfv1::k_encode<true><<<P.tiles_per_part, kThreads, q->smem_k1, s>>>(P, q->ctl);
            return true;
        }
        case 1:
            hwfv1::k_encode_top<true><<<1, kThreads, q->smem_k1, s>>>(P, q->ctl);
            if (P.has_ina) hwfv1::k_ina_mix<<<std::max(1, q->num_sms * 4), kThreads, 0, s>>>(P);
            return true;
        case 2: q->k2<<<P.tiles_per_part, kThreads, q->smem_k2, s>>>(P, q->ctl, 1, 0); return true;
        case 3: q->k3<<<P.tiles_per_part + 1, kThreads, q->smem_k3, s>>>(P, q->ctl, 1, 0ull); return true;
        case 4:
            cudaMemcpyAsync(P.cells[1], P.cells[0], static_cast<size_t>(q->n_cells) * sizeof(double4),
                            cudaMemcpyDeviceToDevice, s);
            hwfv1::k_set_parity<<<1, 32, 0, s>>>(q->ctl, 1);
            hwfv1::k_near_l1<<<q->num_sms * 4, kThreads, 0, s>>>(P, q->ctl);
            hwfv1::k_cfl_init<<<q->fv1_grid, kThreads, 0, s>>>(P, q->ctl, 0);
            return true;
        default: hwfv1::k_finalize<<<1, 32, 0, s>>>(P, q->ctl, 0); return true;
    }
}
constexpr int kInitPhases = 6;

// one partition on its own stream, device barriers between the phases
// (distinct devices / processes)
// (no barrier after the finalize: it reads the peers' CFL slots of this step,
// which they do not touch again before the next step's FV1 barrier, and the
// next K1 reads only this partition's cells)
void part_enqueue_step(swamp_gpu* q) {
    for (int k = 0; k < kStepPhases; ++k)
        if (part_step_phase(q, k, q->stream) && k + 1 < kStepPhases) part_barrier(q, q->stream);
}
void part_enqueue_init(swamp_gpu* q) {
    for (int k = 0; k < kInitPhases; ++k)
        if (part_init_phase(q, k, q->stream)) part_barrier(q, q->stream);
}
// all partitions of a group that share one device: every partition's phase k
// on one stream before phase k + 1 (stream order is the barrier; two streams
// of one context may share a hardware queue, so spinning barriers could
// serialise behind each other)
// Concurrent form (grp->concurrent, the default): phase k of every partition
// on its own stream, forked from and joined back into parts[0]'s stream
// (event edges in the captured graph: the join is the phase barrier, no
// spinning), so the partitions' kernels share the GPU as they would share a
// node's GPUs; each partition's FV1 grid is the device's divided by G.
void serial_enqueue_step(swamp_gpu* grp) {
    cudaStream_t s0 = grp->parts[0]->stream;
    if (!grp->concurrent) {
        for (int k = 0; k < kStepPhases; ++k)
            for (swamp_gpu* q : grp->parts) part_step_phase(q, k, s0);
        return;
    }
    const size_t G = grp->parts.size();
    for (int k = 0; k < kStepPhases; ++k) {
        if (k == 1 && grp->parts[0]->P.top_mode != 2) continue;
        cudaEventRecord(grp->ev_fork, s0);
        for (size_t i = 1; i < G; ++i) cudaStreamWaitEvent(grp->parts[i]->stream, grp->ev_fork, 0);
        for (size_t i = 0; i < G; ++i) part_step_phase(grp->parts[i], k, grp->parts[i]->stream, false);
        for (size_t i = 1; i < G; ++i) {
            cudaEventRecord(grp->ev_join[i], grp->parts[i]->stream);
            cudaStreamWaitEvent(s0, grp->ev_join[i], 0);
        }
    }
}
void serial_enqueue_init(swamp_gpu* grp) {
    for (int k = 0; k < kInitPhases; ++k)
        for (swamp_gpu* q : grp->parts) part_init_phase(q, k, grp->parts[0]->stream);
}

// after initialise: clear the CFL slots / timeline / K3 epochs (the trailing
// barrier guarantees every peer has read this partition's slot)
void part_after_init(swamp_gpu* q) {
    cudaMemsetAsync(q->ctl->rate_bits, 0, sizeof(q->ctl->rate_bits), q->stream);
    cudaMemsetAsync(q->ctl->tl, 0, sizeof(q->ctl->tl), q->stream);
    cudaMemsetAsync(&q->ctl->k3_ready, 0, sizeof(q->ctl->k3_ready), q->stream);
    cudaMemsetAsync(q->P.k3_rec, 0, q->P.n_tiles * 4 * sizeof(unsigned long long), q->stream);
}

// step graphs (graph1 = 1 step, graphS = kGraphSteps) of `g`, captured on
// stream s from `enqueue_step`
template <class F>
int capture_step_graphs(swamp_gpu* g, cudaStream_t s, F&& enqueue_step) {
    for (int which = 0; which < 2; ++which) {
        const int steps = which == 1 ? kGraphSteps : 1;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < steps; ++k) enqueue_step();
        CK(cudaStreamEndCapture(s, &graph));
        if (which == 0) g->launches_per_step = kernel_nodes(graph);
        cudaGraphExec_t exec;
        CK(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        (which == 0 ? g->graph1 : g->graphS) = exec;
    }
    return SWAMP_OK;
}
int part_build_graphs(swamp_gpu* q) {
    return capture_step_graphs(q, q->stream, [&] { part_enqueue_step(q); });
}

int part_enqueue(swamp_gpu* q, int64_t n_steps) {
    swamp_gpu* g = q;
    cudaSetDevice(q->device);
    int64_t k = 0;
    for (; k + kGraphSteps <= n_steps; k += kGraphSteps) CK(cudaGraphLaunch(q->graphS, q->stream));
    for (; k < n_steps; ++k) CK(cudaGraphLaunch(q->graph1, q->stream));
    return SWAMP_OK;
}

int group_sync(swamp_gpu* grp) {
    for (swamp_gpu* q : grp->parts) {
        cudaSetDevice(q->device);
        cudaError_t e = cudaStreamSynchronize(q->stream);
        if (e != cudaSuccess) {
            grp->err = cudaGetErrorString(e);
            return SWAMP_E_CUDA;
        }
    }
    for (swamp_gpu* q : grp->parts) {
        int st = fetch_ctl(q);
        if (st) {
            grp->err = q->err;
            return st;
        }
    }
    return SWAMP_OK;
}

// peer tables of partition q from the partitions' own arrays (one process)
void fill_peer_tables(swamp_gpu* q, const std::vector<swamp_gpu*>& parts) {
    for (size_t k = 0; k < parts.size(); ++k) {
        swamp_gpu* r = parts[k];
        for (int b = 0; b < 2; ++b) {
            q->P.pcells[k][b] = r->P.cells[b];
            q->P.psig[k][b] = r->P.sig[b];
        }
        q->P.ppre[k] = r->P.pre;
        q->P.pdem[k] = r->P.dem;
        q->P.pwet[k][0] = r->P.wet[0];
        q->P.pwet[k][1] = r->P.wet[1];
        q->P.ptile_cnt[k] = r->P.tile_cnt;
        q->P.pctl[k] = r->ctl;
    }
}

int create_group(const swamp_config* cfg, const double* h, const double* qx, const double* qy, const double* z,
                 int G, const int* devices, swamp_gpu** out) {
    if (!out || !h || !qx || !qy || !z || G < 1 || G > hwfv1::kMaxParts) return SWAMP_E_ARG;
    *out = nullptr;
    int st = validate(cfg);
    if (st) return st;
    auto* grp = new swamp_gpu();
    auto fail = [&](int code) {
        delete grp;
        return code;
    };
    grp->device = devices ? devices[0] : 0;
    for (int g = 0; g < G; ++g) {
        auto* q = new swamp_gpu();
        grp->parts.push_back(q);
        if ((st = setup_part(q, cfg, h, qx, qy, z, devices ? devices[g] : 0, G, g))) {
            grp->err = q->err;
            return fail(st);
        }
    }
    // peer access between distinct devices (NVLink / NVSwitch)
    for (int a = 0; a < G; ++a)
        for (int b = 0; b < G; ++b) {
            const int da = grp->parts[a]->device, db = grp->parts[b]->device;
            if (da == db) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, da, db);
            if (!can) return fail(SWAMP_E_CUDA);
            cudaSetDevice(da);
            const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(SWAMP_E_CUDA);
            cudaGetLastError();
        }
    for (swamp_gpu* q : grp->parts) fill_peer_tables(q, grp->parts);
    // one device for all partitions (virtual partitions): one stream, phase
    // order; distinct devices: a stream each, device barriers
    bool same = true, distinct = true;
    for (int a = 0; a < G; ++a)
        for (int b = a + 1; b < G; ++b) {
            same = same && grp->parts[a]->device == grp->parts[b]->device;
            distinct = distinct && grp->parts[a]->device != grp->parts[b]->device;
        }
    if (!same && !distinct) return fail(SWAMP_E_ARG);
    grp->serial = same && G > 1;
    if (grp->serial) {
        cudaSetDevice(grp->parts[0]->device);
        serial_enqueue_init(grp);
    } else {
        for (swamp_gpu* q : grp->parts) {
            cudaSetDevice(q->device);
            part_enqueue_init(q);
        }
    }
    if ((st = group_sync(grp))) return fail(st);
    for (swamp_gpu* q : grp->parts) {
        cudaSetDevice(q->device);
        part_after_init(q);
        if (!grp->serial && (st = part_build_graphs(q))) {
            grp->err = q->err;
            return fail(st);
        }
    }
    if ((st = group_sync(grp))) return fail(st);
    if (grp->serial) {
        cudaSetDevice(grp->parts[0]->device);
        const char* ec = std::getenv("SWAMP_PART_CONCURRENT");
        grp->concurrent = !(ec && ec[0] == '0');
        if (grp->concurrent) {
            bool ok = cudaEventCreateWithFlags(&grp->ev_fork, cudaEventDisableTiming) == cudaSuccess;
            for (int g = 1; g < G; ++g)
                ok = ok && cudaEventCreateWithFlags(&grp->ev_join[g], cudaEventDisableTiming) == cudaSuccess;
            if (!ok) return fail(SWAMP_E_CUDA);
            // the device's FV1 grid shared by the concurrent partitions
            for (swamp_gpu* q : grp->parts) q->fv1_grid = std::max(q->num_sms, q->fv1_grid / G);
        }
        if ((st = capture_step_graphs(grp, grp->parts[0]->stream, [&] { serial_enqueue_step(grp); }))) return fail(st);
    }
    *out = grp;
    return SWAMP_OK;
}

// leaves_x (Morton order, already built) -> host leaves + W/E/N/S descriptors
int copy_leaves_x(swamp_gpu* g, uint32_t N, uint32_t* leaves, uint32_t* nw, uint32_t* ne, uint32_t* nn,
                  uint32_t* ns) {
    cudaSetDevice(g->device);
    if (leaves) CK(cudaMemcpy(leaves, g->P.leaves_x, N * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (nw || ne || nn || ns) {
        uint32_t* d = nullptr;
        CK(cudaMalloc(&d, std::max<size_t>(16, 4ull * N * sizeof(uint32_t))));
        const int grid = std::max(1, std::min<int>(g->num_sms * 8, (N + kThreads - 1) / kThreads));
        hwfv1::k_descriptors<<<grid, kThreads, 0, g->stream>>>(g->P, g->ctl, d, N);
        cudaError_t e = cudaStreamSynchronize(g->stream);
        uint32_t* outs[4] = {nw, ne, nn, ns};
        for (int k = 0; k < 4 && e == cudaSuccess; ++k)
            if (outs[k]) e = cudaMemcpy(outs[k], d + static_cast<size_t>(k) * N, N * sizeof(uint32_t), cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
    }
    return SWAMP_OK;
}

int group_copy_leaves(swamp_gpu* grp, uint32_t* leaves, uint32_t* nw, uint32_t* ne, uint32_t* nn, uint32_t* ns,
                      int64_t cap, int64_t* n) {
    int st = group_sync(grp);
    if (st) return st;
    swamp_gpu* p0 = grp->parts[0];
    const uint32_t N = p0->ctl_host->n_leaves;
    if (n) *n = N;
    if (!leaves && !nw && !ne && !nn && !ns) return SWAMP_OK;
    if (cap < static_cast<int64_t>(N)) return SWAMP_E_ARG;
    for (swamp_gpu* q : grp->parts) {
        cudaSetDevice(q->device);
        q->k3x<<<q->P.tiles_per_part + 1, kThreads, q->smem_k3, q->stream>>>(q->P, q->ctl, 1, ++q->export_epoch);
    }
    if ((st = group_sync(grp))) return st;
    const uint32_t nt = static_cast<uint32_t>(p0->P.n_tiles);
    // each partition's K3 recorded its first subtree's export offset at tile_off[2 nt + tile_lo]
    const size_t G = grp->parts.size();
    std::vector<uint32_t> lo(G + 1, N);
    for (size_t k = 0; k < G; ++k) {
        swamp_gpu* q = grp->parts[k];
        cudaSetDevice(q->device);
        if (cudaMemcpy(&lo[k], q->P.tile_off + 2 * nt + q->P.tile_lo, sizeof(uint32_t), cudaMemcpyDeviceToHost) !=
            cudaSuccess)
            return SWAMP_E_CUDA;
    }
    for (size_t k = 1; k < G; ++k) {  // gather the Morton-ordered slices into partition 0
        swamp_gpu* q = grp->parts[k];
        const uint32_t a = lo[k], b = lo[k + 1];
        if (b > a &&
            cudaMemcpyPeer(p0->P.leaves_x + a, p0->device, q->P.leaves_x + a, q->device, (b - a) * sizeof(uint32_t)) !=
                cudaSuccess)
            return SWAMP_E_CUDA;
    }
    cudaSetDevice(p0->device);
    return copy_leaves_x(p0, N, leaves, nw, ne, nn, ns);
}

int group_advance(swamp_gpu* grp, int64_t n_steps, bool sync, swamp_step_report* rep) {
    if (grp->serial) {
        swamp_gpu* g = grp;
        cudaStream_t s0 = grp->parts[0]->stream;
        cudaSetDevice(grp->parts[0]->device);
        int64_t k = 0;
        for (; k + kGraphSteps <= n_steps; k += kGraphSteps) CK(cudaGraphLaunch(grp->graphS, s0));
        for (; k < n_steps; ++k) CK(cudaGraphLaunch(grp->graph1, s0));
    } else {
        // distinct devices: the partitions meet in device barriers every
        // step, so their launch queues must advance together — round robin,
        // kGraphSteps steps per partition at a time (queuing all of one
        // partition's steps first could fill its launch queue and block the
        // host while that device spins on a peer with nothing queued)
        for (int64_t k = 0; k < n_steps; k += kGraphSteps) {
            const int64_t chunk = std::min<int64_t>(kGraphSteps, n_steps - k);
            for (swamp_gpu* q : grp->parts) {
                const int st = part_enqueue(q, chunk);
                if (st) {
                    grp->err = q->err;
                    return st;
                }
            }
        }
    }
    if (!sync) return SWAMP_OK;
    int st = group_sync(grp);
    fill_group_report(grp, rep);
    return st;
}

// ---- dynamic repartitioning: contiguous subtree ranges
// that equalise the leaf counts, from the per-subtree list offsets K3's top
// CTA wrote (every partition holds them for all subtrees)
// contiguous subtree ranges [nb[g], nb[g+1]) with ~equal leaf counts from the
// cumulative counts before[t] (t = 0..nt; before[nt] = all leaves); boundary
// granularity 16 subtrees when there are plenty (keeps K3's 16-byte staging),
// finer for small grids; every partition keeps at least that many subtrees.
// The same function serves swamp_partition_plan (host, no device).
void plan_bounds_host(uint32_t nt, int G, const uint64_t* before, uint32_t* nb) {
    const uint64_t N = before[nt];
    const uint32_t al = (nt >= 64u * G) ? 16u : (nt >= 16u * G) ? 4u : 1u;
    nb[0] = 0;
    for (int g = 1; g < G; ++g) {
        const uint64_t target = N * static_cast<uint64_t>(g) / G;
        uint32_t t = nb[g - 1] + al;
        while (t + al * static_cast<uint32_t>(G - g) <= nt && before[t] < target) t += al;
        if (t + al * static_cast<uint32_t>(G - g) > nt) t = nt - al * static_cast<uint32_t>(G - g);
        nb[g] = t;
    }
    for (int g = G; g <= hwfv1::kMaxParts; ++g) nb[g] = nt;
}

bool plan_bounds(swamp_gpu* q, int G, uint32_t* nb) {
    const uint32_t nt = static_cast<uint32_t>(q->P.n_tiles);
    std::vector<uint32_t> off(2 * static_cast<size_t>(nt));
    if (cudaMemcpy(off.data(), q->P.tile_off, off.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
        return false;
    const uint64_t ta = q->ctl_host->n_leaves_A, N = q->ctl_host->n_leaves;
    std::vector<uint64_t> before(static_cast<size_t>(nt) + 1);
    for (uint32_t t = 0; t < nt; ++t) before[t] = static_cast<uint64_t>(off[t]) + off[nt + t] - ta;  // leaves of [0, t)
    before[nt] = N;
    plan_bounds_host(nt, G, before.data(), nb);
    return true;
}

void apply_bounds(Params& P, const uint32_t* nb) {
    for (int k = 0; k <= hwfv1::kMaxParts; ++k) P.pbound[k] = nb[k];
    P.tile_lo = nb[P.part];
    P.tile_hi = nb[P.part + 1];
    P.tiles_per_part = P.tile_hi - P.tile_lo;
    uint32_t a = 16;
    for (int k = 0; k <= P.G; ++k) {
        while (a > 1 && nb[k] % a) a = (a == 16) ? 4 : 1;
    }
    P.pb_align = a;
}

// ---- one partition per process (rank engines)
struct RankBlob {  // exchanged between the ranks (swamp_gpu_rank_create / _connect)
    uint32_t magic;
    int32_t rank, world, device;
    uint64_t pid;
    uint64_t ptr[10];             // cells[0], cells[1], sig[0], sig[1], pre, tile_cnt, ctl, dem, wet[0], wet[1]
    cudaIpcMemHandle_t ipc[10];
};
static_assert(sizeof(RankBlob) <= SWAMP_RANK_BLOB_BYTES, "rank blob too large");
constexpr uint32_t kRankMagic = 0x53574D52u;  // "SWMR"

void* rank_ptr(const swamp_gpu* q, int k) {
    switch (k) {
        case 0: return q->P.cells[0];
        case 1: return q->P.cells[1];
        case 2: return q->P.sig[0];
        case 3: return q->P.sig[1];
        case 4: return q->P.pre;
        case 5: return q->P.tile_cnt;
        case 6: return q->ctl;
        case 7: return q->P.dem;
        case 8: return q->P.wet[0];
        default: return q->P.wet[1];
    }
}

}  // namespace

extern "C" {

int swamp_gpu_create(const swamp_config* cfg, const double* h, const double* qx, const double* qy, const double* z,
                     int device, swamp_gpu** out) {
    return create_impl(cfg, h, qx, qy, z, device, false, out);
}

int swamp_gpu_create_uniform(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                             const double* z, int device, swamp_gpu** out) {
    return create_impl(cfg, h, qx, qy, z, device, true, out);
}

int swamp_gpu_trim_cache(int device) {
    BlockCache& c = block_cache();
    std::vector<std::pair<int, void*>> dev;
    std::vector<void*> pinned;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.dev.begin(); it != c.dev.end();) {
            if (device < 0 || it->first.first == device) {
                dev.push_back({it->first.first, it->second});
                c.bytes -= it->first.second;
                it = c.dev.erase(it);
            } else {
                ++it;
            }
        }
        if (device < 0) pinned.swap(c.pinned);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& d : dev) {
        cudaSetDevice(d.first);
        cudaFree(d.second);
    }
    cudaSetDevice(cur);
    for (void* p : pinned) cudaFreeHost(p);
    return SWAMP_OK;
}

int swamp_gpu_destroy(swamp_gpu* g) {
    if (!g) return SWAMP_E_ARG;
    cudaSetDevice(g->device);
    delete g;
    return SWAMP_OK;
}

int swamp_gpu_set_profiling(swamp_gpu* g, int enabled) {
    if (!g) return SWAMP_E_ARG;
    g->profiling = enabled != 0;
    return SWAMP_OK;
}

int swamp_gpu_create_partitioned(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                                 const double* z, int n_parts, const int* devices, swamp_gpu** out) {
    return create_group(cfg, h, qx, qy, z, n_parts, devices, out);
}

int swamp_gpu_step(swamp_gpu* g, swamp_step_report* rep) {
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) return group_advance(g, 1, true, rep);
    cudaSetDevice(g->device);
    // fast path: the step's FV1 writes the control block into the pinned
    // mirror; the host waits for its sequence word instead of copying and
    // synchronising (falls back to the copy if the word does not arrive)
    if (g->P.ctl_mirror && g->graphR && !g->profiling && !g->uniform && g->mirror_current &&
        g->ctl_host->t < g->P.t_end) {
        volatile unsigned long long* seq = &g->ctl_host->rep_seq;
        const unsigned long long expect = static_cast<unsigned long long>(g->ctl_host->step) + 1ull;
        g->mirror_current = false;
        CK(cudaGraphLaunch(g->graphR, g->stream));
        const auto t0 = std::chrono::steady_clock::now();
        bool arrived = false;
        for (unsigned spin = 0;; ++spin) {
            if (*seq == expect) {
                arrived = true;
                std::atomic_thread_fence(std::memory_order_acquire);  // the report words before rep_seq
                break;
            }
            if ((spin & 1023u) == 1023u &&
                std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(200))
                break;
        }
        if (arrived && g->ctl_host->err_code == 0) {
            g->mirror_current = true;
            fill_report(g, rep);
            return SWAMP_OK;
        }
        const int st = fetch_ctl(g);  // error or no word: the synchronous path decides
        fill_report(g, rep);
        return st;
    }
    if (g->profiling && g->rank_world == 0 && ensure_graph(g, 2) == SWAMP_OK && g->graphT) {
        CK(cudaGraphLaunch(g->graphT, g->stream));
    } else {
        CK(cudaGraphLaunch(g->graph1, g->stream));
    }
    int st = fetch_ctl(g);
    fill_report(g, rep);
    if (rep && g->profiling) {
        float ms[4] = {0, 0, 0, 0};
        for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms[k], g->ev[k], g->ev[k + 1]);
        rep->ms_encode_flag = ms[0];
        rep->ms_band_closure = ms[1];
        rep->ms_decode_traverse = ms[2];
        rep->ms_neighbours = 0.0;
        rep->ms_fv1 = ms[3];
        float tot = 0;
        cudaEventElapsedTime(&tot, g->ev[0], g->ev[4]);
        rep->ms_total = tot;
    }
    return st;
}

int swamp_gpu_stream(swamp_gpu* g, void** stream) {
    if (!g || !stream) return SWAMP_E_ARG;
    if (!g->parts.empty()) g = g->parts[0];
    *stream = static_cast<void*>(g->stream);
    return SWAMP_OK;
}

int swamp_gpu_enqueue(swamp_gpu* g, int64_t n_steps) {
    if (!g || n_steps < 0) return SWAMP_E_ARG;
    if (!g->parts.empty()) return group_advance(g, n_steps, false, nullptr);
    cudaSetDevice(g->device);
    if (n_steps > 0) g->mirror_current = false;  // (the mirror moves on asynchronously)
    int64_t k = 0;
    if (n_steps >= kGraphSteps) {
        const int st = ensure_graph(g, 1);
        if (st) return st;
    }
    for (; k + kGraphSteps <= n_steps; k += kGraphSteps) CK(cudaGraphLaunch(g->graphS, g->stream));
    for (; k < n_steps; ++k) CK(cudaGraphLaunch(g->graph1, g->stream));
    return SWAMP_OK;
}

int swamp_gpu_advance(swamp_gpu* g, int64_t n_steps, swamp_step_report* rep) {
    if (!g || n_steps < 0) return SWAMP_E_ARG;
    if (!g->parts.empty()) return group_advance(g, n_steps, true, rep);
    cudaSetDevice(g->device);
    int64_t k = 0;
    if (n_steps >= kGraphSteps) {
        const int st = ensure_graph(g, 1);
        if (st) return st;
    }
    for (; k + kGraphSteps <= n_steps; k += kGraphSteps) CK(cudaGraphLaunch(g->graphS, g->stream));
    for (; k < n_steps; ++k) CK(cudaGraphLaunch(g->graph1, g->stream));
    int st = fetch_ctl(g);
    fill_report(g, rep);
    return st;
}

// n steps back to back, every step's report read into host memory as the
// step completes (the step's finalize writes it into a pinned ring slot;
// the host copies each out while later steps run, at most kRepRing steps
// ahead of it). Steps past t_end are device-side no-ops: their reports
// repeat the final state.
int swamp_gpu_advance_reports(swamp_gpu* g, int64_t n_steps, swamp_step_report* reps) {
    if (!g || n_steps < 0 || (n_steps > 0 && !reps)) return SWAMP_E_ARG;
    if (n_steps == 0) return SWAMP_OK;
    const bool ring = g->parts.empty() && g->ring_dev && !g->uniform && !g->profiling && g->rank_world == 0;
    if (!ring) {  // partitions, ranks, uniform, profiling: one synchronising step per report
        for (int64_t k = 0; k < n_steps; ++k) {
            const int st = swamp_gpu_step(g, &reps[k]);
            if (st) return st;
        }
        return SWAMP_OK;
    }
    cudaSetDevice(g->device);
    int st = SWAMP_OK;
    if (!g->mirror_current && (st = fetch_ctl(g))) return st;
    if ((st = ensure_graph(g, 4)) || (st = ensure_graph(g, 5))) return st;
    Ctl* const ring_host = g->ctl_host + 1;
    // (the pinned block may come from the process cache: no stale sequence words)
    for (int k = 0; k < kRepRing; ++k) *reinterpret_cast<volatile unsigned long long*>(&ring_host[k].rep_seq) = ~0ull;
    const unsigned long long step0 = static_cast<unsigned long long>(g->ctl_host->step);
    bool ended = !(g->ctl_host->t < g->P.t_end);
    int64_t launched = 0, done = 0;
    g->mirror_current = false;
    while (done < n_steps) {
        if (!ended)
            while (launched < n_steps) {
                const int64_t b = (n_steps - launched >= kGraphSteps) ? kGraphSteps : 1;
                if (launched + b - done > kRepRing) break;
                CK(cudaGraphLaunch(b == kGraphSteps ? g->graphQ : g->graphQ1, g->stream));
                launched += b;
            }
        if (ended) {  // no-op steps: the final state
            if ((st = fetch_ctl(g))) return st;
            for (; done < n_steps; ++done) fill_report(g, &reps[done]);
            return SWAMP_OK;
        }
        if (done == n_steps - 1) {  // the last step's report: no later K1 writes it
            if ((st = fetch_ctl(g))) return st;
            fill_report(g, &reps[done]);
            ++done;
            continue;
        }
        const unsigned long long expect = step0 + static_cast<unsigned long long>(done) + 1ull;
        const Ctl& c = ring_host[expect & (kRepRing - 1)];
        volatile const unsigned long long* seq = &c.rep_seq;
        const auto t0 = std::chrono::steady_clock::now();
        for (unsigned spin = 0;; ++spin) {
            if (*seq == expect) break;
            if ((spin & 255u) == 255u) {
                // the stream drained without this report: the step was a no-op
                // (t reached t_end) — unless the word landed meanwhile
                if (cudaStreamQuery(g->stream) == cudaSuccess && *seq != expect) {
                    ended = true;
                    break;
                }
                if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(10)) return SWAMP_E_CUDA;
            }
        }
        if (ended) continue;
        std::atomic_thread_fence(std::memory_order_acquire);  // the report words before rep_seq
        if (c.err_code != 0) {
            st = fetch_ctl(g);
            fill_report(g, &reps[done]);
            return st ? st : SWAMP_E_NONFINITE;
        }
        fill_report_from(g, c, &reps[done]);
        ++done;
    }
    return fetch_ctl(g);
}

int swamp_gpu_step_uniform(swamp_gpu* g, int64_t n_steps, swamp_step_report* rep) {
    if (!g || !g->uniform) return SWAMP_E_STATE;
    return swamp_gpu_advance(g, n_steps, rep);
}

int swamp_gpu_run(swamp_gpu* g, swamp_step_report* rep) {
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) {
        int st = group_sync(g);
        if (st) return st;
        while (g->parts[0]->ctl_host->t < g->parts[0]->P.t_end)
            if ((st = group_advance(g, 16, true, rep))) return st;
        fill_group_report(g, rep);
        return SWAMP_OK;
    }
    int st = fetch_ctl(g);
    if (st) return st;
    while (g->ctl_host->t < g->P.t_end) {
        st = swamp_gpu_advance(g, 64, rep);
        if (st) return st;
    }
    fill_report(g, rep);
    return SWAMP_OK;
}

int swamp_gpu_info(const swamp_gpu* gc, double* t, double* dt, int64_t* step, int64_t* n_leaves) {
    swamp_gpu* g = const_cast<swamp_gpu*>(gc);
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) {
        const int st = group_sync(g);
        if (st) return st;
        g = g->parts[0];
    }
    cudaSetDevice(g->device);
    int st = fetch_ctl(g);
    if (t) *t = g->ctl_host->t;
    if (dt) *dt = g->ctl_host->dt;
    if (step) *step = g->ctl_host->step;
    if (n_leaves) *n_leaves = g->uniform ? (int64_t(1) << (2 * g->P.L)) : g->ctl_host->n_leaves;
    return st;
}

int swamp_gpu_copy_leaves(swamp_gpu* g, uint32_t* leaves, uint32_t* nw, uint32_t* ne, uint32_t* nn, uint32_t* ns,
                          int64_t cap, int64_t* n) {
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) return group_copy_leaves(g, leaves, nw, ne, nn, ns, cap, n);
    cudaSetDevice(g->device);
    int st = fetch_ctl(g);
    if (st) return st;
    const uint32_t N = g->ctl_host->n_leaves;
    if (n) *n = N;
    if (!leaves && !nw && !ne && !nn && !ns) return SWAMP_OK;
    if (g->rank_world > 1) return SWAMP_E_STATE;  // a rank holds only its own slice: count only
    if (cap < static_cast<int64_t>(N)) return SWAMP_E_ARG;
    // Morton-ordered LeafAssembly of the current tree (the hot path keeps the
    // level-L leaves first)
    g->k3x<<<g->P.n_tiles + 1, kThreads, g->smem_k3, g->stream>>>(g->P, g->ctl, 1, ++g->export_epoch);
    CK(cudaStreamSynchronize(g->stream));
    return copy_leaves_x(g, N, leaves, nw, ne, nn, ns);
}

int swamp_gpu_export_tree(swamp_gpu* g, double* h, double* qx, double* qy, double* z, uint8_t* sig) {
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) {  // owner-aware export from partition 0
        const int st = group_sync(g);
        if (st) return st;
        g = g->parts[0];
    }
    cudaSetDevice(g->device);
    const size_t NH = swamp::zorder::hierarchy_cells(g->P.L);
    const size_t ND = swamp::zorder::detail_cells(g->P.L);
    double* d = nullptr;
    uint8_t* ds = nullptr;
    CK(cudaMalloc(&d, 4 * NH * sizeof(double)));
    cudaError_t e = cudaMalloc(&ds, std::max<size_t>(ND, 16));
    if (e == cudaSuccess) {
        hwfv1::k_export_tree<<<std::max(1, g->num_sms * 8), kThreads, 0, g->stream>>>(g->P, g->ctl, d, d + NH,
                                                                                       d + 2 * NH, d + 3 * NH, ds);
        e = cudaStreamSynchronize(g->stream);
    }
    double* outs[4] = {h, qx, qy, z};
    for (int q = 0; q < 4 && e == cudaSuccess; ++q)
        if (outs[q]) e = cudaMemcpy(outs[q], d + q * NH, NH * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && sig) e = cudaMemcpy(sig, ds, ND, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (ds) cudaFree(ds);
    CK(e);
    return SWAMP_OK;
}

int swamp_gpu_export_finest(swamp_gpu* g, double* h, double* qx, double* qy) {
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) {
        const int st = group_sync(g);
        if (st) return st;
        g = g->parts[0];
    }
    cudaSetDevice(g->device);
    const size_t nf = static_cast<size_t>(1) << (2 * g->P.L);
    if (!g->scratch) {  // kept for later exports
        CK(cached_malloc(g->device, &g->scratch, 3 * nf * sizeof(double)));
        g->scratch_bytes = 3 * nf * sizeof(double);
    }
    double* d = static_cast<double*>(g->scratch);
    hwfv1::k_export_finest<<<std::max(1, g->num_sms * 8), kThreads, 0, g->stream>>>(g->P, g->ctl, d, d + nf,
                                                                                     d + 2 * nf);
    // async copies on the engine stream: full speed into pinned host buffers
    double* outs[3] = {h, qx, qy};
    for (int q = 0; q < 3; ++q)
        if (outs[q]) CK(cudaMemcpyAsync(outs[q], d + q * nf, nf * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return SWAMP_OK;
}

int swamp_gpu_sample_gauges(swamp_gpu* g, int32_t n, const double* x, const double* y, double* out) {
    if (!g || n < 0 || (n > 0 && (!x || !y || !out))) return SWAMP_E_ARG;
    if (n == 0) return SWAMP_OK;
    if (!g->parts.empty()) {
        const int st = group_sync(g);
        if (st) return st;
        g = g->parts[0];
    }
    const uint32_t side = 1u << g->P.L;
    std::vector<uint32_t> cells(static_cast<size_t>(n));
    for (int32_t k = 0; k < n; ++k) {  // the finest cell whose closed-open square holds the point
        const double fi = std::floor((x[k] - g->x0) / g->P.W * side), fj = std::floor((y[k] - g->y0) / g->P.W * side);
        if (!(fi >= 0.0 && fi < side && fj >= 0.0 && fj < side)) {
            g->err = "gauge " + std::to_string(k) + " outside the domain";
            return SWAMP_E_ARG;
        }
        cells[static_cast<size_t>(k)] = static_cast<uint32_t>(fi) | (static_cast<uint32_t>(fj) << 16);
    }
    cudaSetDevice(g->device);
    void* d = nullptr;
    const size_t cb = (cells.size() * sizeof(uint32_t) + 15) & ~size_t(15), ob = 4 * static_cast<size_t>(n) * sizeof(double);
    CK(cudaMallocAsync(&d, cb + ob, g->stream));
    uint32_t* dc = static_cast<uint32_t*>(d);
    double* dout = reinterpret_cast<double*>(static_cast<char*>(d) + cb);
    cudaError_t e = cudaMemcpyAsync(dc, cells.data(), cells.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, g->stream);
    if (e == cudaSuccess) {
        hwfv1::k_gauges<<<std::max(1, std::min(g->num_sms, (n + kThreads - 1) / kThreads)), kThreads, 0, g->stream>>>(
            g->P, g->ctl, dc, n, dout);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, ob, cudaMemcpyDeviceToHost, g->stream);
    cudaFreeAsync(d, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    CK(e);
    return SWAMP_OK;
}

int swamp_gpu_last_error(const swamp_gpu* g, int32_t* code, uint32_t* z, int32_t* quantity, int32_t* stage, char* msg,
                         size_t msg_cap) {
    if (!g) return SWAMP_E_ARG;
    if (!g->parts.empty()) {
        for (const swamp_gpu* q : g->parts)
            if (q->ctl_host && q->ctl_host->err_code) return swamp_gpu_last_error(q, code, z, quantity, stage, msg, msg_cap);
        if (msg && msg_cap) {
            std::strncpy(msg, g->err.c_str(), msg_cap - 1);
            msg[msg_cap - 1] = 0;
        }
        if (code) *code = 0;
        return SWAMP_OK;
    }
    if (code) *code = g->ctl_host ? g->ctl_host->err_code : 0;
    if (z) *z = g->ctl_host ? g->ctl_host->err_z : 0;
    if (quantity) *quantity = g->ctl_host ? g->ctl_host->err_q : 0;
    if (stage) *stage = g->ctl_host ? g->ctl_host->err_stage : 0;
    if (msg && msg_cap) {
        std::strncpy(msg, g->err.c_str(), msg_cap - 1);
        msg[msg_cap - 1] = 0;
    }
    return SWAMP_OK;
}

int swamp_gpu_timeline(swamp_gpu* g, double* out12) {
    if (!g || !out12) return SWAMP_E_ARG;
    if (!g->parts.empty()) g = g->parts[0];
    int st = fetch_ctl(g);
    // the last completed step ran with step counter (step - 1)
    const auto& tl = g->ctl_host->tl[(g->ctl_host->step - 1) & 1];
    const unsigned long long t0 = ~tl[0][0];
    for (int k = 0; k < 12; ++k) {
        const unsigned long long raw = tl[k / 3][k % 3];
        const unsigned long long v = (k % 3 == 0) ? ~raw : raw;
        out12[k] = (raw == 0 || v < t0) ? -1.0 : 1e-3 * static_cast<double>(v - t0);
    }
    // [1]: the previous step's end relative to this step's K1 start (<= 0)
    out12[1] = (tl[0][1] == 0 || t0 == ~0ull) ? 0.0 : -1e-3 * static_cast<double>(static_cast<long long>(t0 - tl[0][1]));
    return st;
}

int swamp_gpu_debug(swamp_gpu* g, uint64_t* out64) {
    if (!g || !out64) return SWAMP_E_ARG;
    if (!g->parts.empty()) g = g->parts[0];
    int st = fetch_ctl(g);
    std::memcpy(out64, g->ctl_host->dbg, sizeof(g->ctl_host->dbg));
    return st;
}

int swamp_gpu_counters(swamp_gpu* g, int64_t* out8) {
    if (!g || !out8) return SWAMP_E_ARG;
    if (!g->parts.empty()) {
        int64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (swamp_gpu* q : g->parts) {
            int64_t c[8];
            const int st = swamp_gpu_counters(q, c);
            if (st) return st;
            for (int k = 1; k < 3; ++k) acc[k] += c[k];
            acc[6] += c[6];
            acc[7] += c[7];
            acc[5] += c[5];
            acc[0] = c[0];
            acc[3] = c[3];
            acc[4] = c[4];  // global leaf counts: every partition holds the same sum
        }
        if (g->launches_per_step) acc[5] = g->launches_per_step;  // one graph for the whole group
        std::memcpy(out8, acc, sizeof(acc));
        return SWAMP_OK;
    }
    int st = fetch_ctl(g);
    out8[0] = g->uniform ? (int64_t(1) << (2 * g->P.L)) : g->ctl_host->n_leaves_used;
    out8[1] = static_cast<int64_t>(g->ctl_host->cnt_tree);
    out8[2] = static_cast<int64_t>(g->ctl_host->cnt_new);
    out8[3] = int64_t(1) << (2 * g->P.L);
    out8[4] = static_cast<int64_t>(g->ctl_host->cnt_updates);
    out8[5] = g->launches_per_step;  // this engine's kernels per step (one-step graph)
    out8[6] = static_cast<int64_t>(g->ctl_host->cnt_near);
    out8[7] = static_cast<int64_t>(g->ctl_host->near_last);
    return st;
}

int swamp_gpu_skip_counters(swamp_gpu* g, int64_t* out2) {
    if (!g || !out2) return SWAMP_E_ARG;
    out2[0] = out2[1] = 0;
    std::vector<swamp_gpu*> parts = g->parts.empty() ? std::vector<swamp_gpu*>{g} : g->parts;
    if (!g->parts.empty()) {
        const int st = group_sync(g);
        if (st) return st;
    }
    for (swamp_gpu* q : parts) {
        if (g->parts.empty()) {
            cudaSetDevice(q->device);
            const int st = fetch_ctl(q);
            if (st) return st;
        }
        out2[0] += static_cast<int64_t>(q->ctl_host->cnt_skip);
        out2[1] += static_cast<int64_t>(q->ctl_host->cnt_k1skip);
    }
    return SWAMP_OK;
}

int swamp_gpu_work_counters(swamp_gpu* g, int64_t* out8) {
    if (!g || !out8) return SWAMP_E_ARG;
    int64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::vector<swamp_gpu*> parts = g->parts.empty() ? std::vector<swamp_gpu*>{g} : g->parts;
    if (!g->parts.empty()) {
        const int st = group_sync(g);
        if (st) return st;
    }
    for (swamp_gpu* q : parts) {
        if (g->parts.empty()) {
            cudaSetDevice(q->device);
            const int st = fetch_ctl(q);
            if (st) return st;
        }
        const Ctl& c = *q->ctl_host;
        acc[0] += static_cast<int64_t>(c.cnt_tree);
        acc[1] += static_cast<int64_t>(c.cnt_fused);
        acc[2] += static_cast<int64_t>(c.cnt_new);
        acc[3] = static_cast<int64_t>(c.cnt_updates);  // global leaf counts: every partition holds the same sum
        acc[4] += static_cast<int64_t>(c.cnt_quiet);
        acc[5] += static_cast<int64_t>(c.cnt_tiled);
        acc[6] = c.step;
    }
    acc[7] = static_cast<int64_t>(swamp::zorder::detail_cells(g->parts.empty() ? g->P.L : g->parts[0]->P.L));
    std::memcpy(out8, acc, sizeof(acc));
    return SWAMP_OK;
}

int swamp_gpu_near_threshold(swamp_gpu* g, int64_t* out4) {
    if (!g || !out4) return SWAMP_E_ARG;
    int64_t acc[4] = {0, 0, 0, 0};
    std::vector<swamp_gpu*> parts = g->parts.empty() ? std::vector<swamp_gpu*>{g} : g->parts;
    if (!g->parts.empty()) {
        const int st = group_sync(g);
        if (st) return st;
    }
    for (swamp_gpu* q : parts) {
        if (g->parts.empty()) {
            cudaSetDevice(q->device);
            const int st = fetch_ctl(q);
            if (st) return st;
        }
        acc[0] += static_cast<int64_t>(q->ctl_host->near_last);
        acc[1] += static_cast<int64_t>(q->ctl_host->cnt_near);
        acc[2] += static_cast<int64_t>(q->ctl_host->near_init);
        acc[3] += static_cast<int64_t>(q->ctl_host->near_dem);
    }
    std::memcpy(out4, acc, sizeof(acc));
    return SWAMP_OK;
}

int swamp_gpu_rank_create(const swamp_config* cfg, const double* h, const double* qx, const double* qy,
                          const double* z, int rank, int world, int device, swamp_gpu** out, uint8_t* blob) {
    if (!out || !blob || !h || !qx || !qy || !z || world < 1 || world > hwfv1::kMaxParts || rank < 0 || rank >= world)
        return SWAMP_E_ARG;
    *out = nullptr;
    int st = validate(cfg);
    if (st) return st;
    auto* g = new swamp_gpu();
    if ((st = setup_part(g, cfg, h, qx, qy, z, device, world, rank))) {
        delete g;
        return st;
    }
    g->rank_world = world;
    RankBlob b{};
    b.magic = kRankMagic;
    b.rank = rank;
    b.world = world;
    b.device = device;
    b.pid = static_cast<uint64_t>(getpid());
    for (int k = 0; k < 10; ++k) {
        void* p = rank_ptr(g, k);
        b.ptr[k] = reinterpret_cast<uint64_t>(p);
        if (cudaIpcGetMemHandle(&b.ipc[k], p) != cudaSuccess) {
            delete g;
            return SWAMP_E_CUDA;
        }
    }
    std::memset(blob, 0, SWAMP_RANK_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof(b));
    *out = g;
    return SWAMP_OK;
}

int swamp_gpu_rank_connect(swamp_gpu* g, const uint8_t* blobs) {
    if (!g || !blobs || g->rank_world < 1) return SWAMP_E_ARG;
    cudaSetDevice(g->device);
    const int W = g->rank_world, me = g->P.part;
    const uint64_t pid = static_cast<uint64_t>(getpid());
    for (int r = 0; r < W; ++r) {
        RankBlob b;
        std::memcpy(&b, blobs + static_cast<size_t>(r) * SWAMP_RANK_BLOB_BYTES, sizeof(b));
        if (b.magic != kRankMagic || b.rank != r || b.world != W) return SWAMP_E_ARG;
        void* p[10];
        if (r == me) {
            for (int k = 0; k < 10; ++k) p[k] = rank_ptr(g, k);
        } else if (b.pid == pid) {  // another rank handle of this process: its pointers directly
            if (b.device != g->device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return SWAMP_E_CUDA;
                cudaGetLastError();
            }
            for (int k = 0; k < 10; ++k) p[k] = reinterpret_cast<void*>(b.ptr[k]);
        } else {  // another process: open its CUDA IPC handles (NVLink peer mapping)
            for (int k = 0; k < 10; ++k) {
                if (cudaIpcOpenMemHandle(&p[k], b.ipc[k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    g->err = "cudaIpcOpenMemHandle failed";
                    return SWAMP_E_CUDA;
                }
                g->ipc_opened.push_back(p[k]);
            }
        }
        g->P.pcells[r][0] = static_cast<double4*>(p[0]);
        g->P.pcells[r][1] = static_cast<double4*>(p[1]);
        g->P.psig[r][0] = static_cast<uint8_t*>(p[2]);
        g->P.psig[r][1] = static_cast<uint8_t*>(p[3]);
        g->P.ppre[r] = static_cast<uint8_t*>(p[4]);
        g->P.ptile_cnt[r] = static_cast<uint32_t*>(p[5]);
        g->P.pctl[r] = static_cast<Ctl*>(p[6]);
        g->P.pdem[r] = static_cast<uint8_t*>(p[7]);
        g->P.pwet[r][0] = static_cast<uint8_t*>(p[8]);
        g->P.pwet[r][1] = static_cast<uint8_t*>(p[9]);
    }
    part_enqueue_init(g);  // completes once every rank has connected (device barriers)
    return cudaGetLastError() == cudaSuccess ? SWAMP_OK : SWAMP_E_CUDA;
}

int swamp_gpu_rank_ready(swamp_gpu* g) {
    if (!g || g->rank_world < 1) return SWAMP_E_ARG;
    cudaSetDevice(g->device);
    int st = fetch_ctl(g);
    if (st) return st;
    part_after_init(g);
    if ((st = part_build_graphs(g))) return st;
    return fetch_ctl(g);
}

int swamp_gpu_compare(swamp_gpu* a, swamp_gpu* b, double* l1, double* linf) {
    if (!a || !b || !l1 || !linf) return SWAMP_E_ARG;
    swamp_gpu* ga = a->parts.empty() ? a : a->parts[0];
    swamp_gpu* gb = b->parts.empty() ? b : b->parts[0];
    if (ga->P.L != gb->P.L || ga->P.W != gb->P.W) return SWAMP_E_ARG;  // mismatched grids
    if (ga->device != gb->device) return SWAMP_E_ARG;
    if (!a->parts.empty() && group_sync(a)) return SWAMP_E_CUDA;
    if (!b->parts.empty() && group_sync(b)) return SWAMP_E_CUDA;
    swamp_gpu* g = ga;
    cudaSetDevice(ga->device);
    const size_t nf = static_cast<size_t>(1) << (2 * ga->P.L);
    const int blocks = std::max(1, std::min<int>(ga->num_sms * 4, static_cast<int>((nf + kThreads - 1) / kThreads)));
    double* d = nullptr;
    CK(cudaMalloc(&d, (6 * nf + 2 * blocks) * sizeof(double)));
    cudaStreamSynchronize(gb->stream);
    hwfv1::k_export_finest<<<std::max(1, ga->num_sms * 8), kThreads, 0, ga->stream>>>(ga->P, ga->ctl, d, d + nf, d + 2 * nf);
    hwfv1::k_export_finest<<<std::max(1, ga->num_sms * 8), kThreads, 0, ga->stream>>>(gb->P, gb->ctl, d + 3 * nf,
                                                                                       d + 4 * nf, d + 5 * nf);
    hwfv1::k_compare<<<blocks, kThreads, 0, ga->stream>>>(d, d + 3 * nf, nf, d + 6 * nf, d + 6 * nf + blocks);
    std::vector<double> part(2 * static_cast<size_t>(blocks));
    cudaError_t e = cudaMemcpyAsync(part.data(), d + 6 * nf, part.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                    ga->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ga->stream);
    cudaFree(d);
    CK(e);
    double s = 0.0, m = 0.0;
    for (int k = 0; k < blocks; ++k) {
        s += part[k];
        m = std::max(m, part[blocks + k]);
    }
    *l1 = s / static_cast<double>(nf);  // sum |dh| dx^2 / area over the square: the mean
    *linf = m;
    return SWAMP_OK;
}

int swamp_partition_plan(int32_t L, int32_t G, const uint64_t* leaves_before, uint32_t* bounds) {
    if (L < 1 || L > 13 || G < 1 || G > hwfv1::kMaxParts || !bounds) return SWAMP_E_ARG;
    const int R = L - std::min(L, 6);
    const uint32_t nt = 1u << (2 * R);
    if (nt % static_cast<uint32_t>(G) != 0) return SWAMP_E_ARG;
    uint32_t nb[hwfv1::kMaxParts + 1];
    if (leaves_before) {
        for (uint32_t t = 0; t < nt; ++t)
            if (leaves_before[t + 1] < leaves_before[t]) return SWAMP_E_ARG;
        plan_bounds_host(nt, G, leaves_before, nb);
    } else {  // the creation plan: equal subtree counts
        for (int g = 0; g <= hwfv1::kMaxParts; ++g) nb[g] = static_cast<uint32_t>(std::min(g, G)) * (nt / G);
    }
    for (int g = 0; g <= G; ++g) bounds[g] = nb[g];
    return SWAMP_OK;
}

int swamp_partition_owner(const uint32_t* bounds, int32_t G, int32_t L, int32_t n, uint32_t m) {
    if (!bounds || G < 1 || G > hwfv1::kMaxParts || L < 1 || L > 13 || n < 0 || n > L) return SWAMP_E_ARG;
    if (m >= (1u << (2 * n))) return SWAMP_E_ARG;
    const int R = L - std::min(L, 6);
    return hwfv1::owner_in(bounds, G, R, n, m);
}

int swamp_gpu_rebalance(swamp_gpu* g, int32_t* changed) {
    if (!g) return SWAMP_E_ARG;
    if (changed) *changed = 0;
    const bool group = !g->parts.empty();
    if (!group && g->rank_world < 2) return SWAMP_OK;  // one partition: nothing to balance
    int st = group ? group_sync(g) : fetch_ctl(g);
    if (st) return st;
    std::vector<swamp_gpu*> mine = group ? g->parts : std::vector<swamp_gpu*>{g};
    swamp_gpu* q0 = mine[0];
    const int G = q0->P.G;
    uint32_t nb[hwfv1::kMaxParts + 1];
    cudaSetDevice(q0->device);
    if (!plan_bounds(q0, G, nb)) return SWAMP_E_CUDA;
    bool same = true;
    for (int k = 0; k <= G; ++k) same = same && nb[k] == q0->P.pbound[k];
    if (same) return SWAMP_OK;
    // every partition pulls what it gains from the old owners (peers idle: a
    // rank engine first meets its peers on the device)
    std::vector<Params> old;
    for (swamp_gpu* q : mine) old.push_back(q->P);
    for (size_t k = 0; k < mine.size(); ++k) {
        swamp_gpu* q = mine[k];
        cudaSetDevice(q->device);
        if (!group) part_barrier(q, q->stream);
        Params np = q->P;
        apply_bounds(np, nb);
        cudaStream_t s = (group && g->serial) ? q0->stream : q->stream;
        if (np.tiles_per_part > 0) hwfv1::k_rebalance_pull<<<np.tiles_per_part, kThreads, 0, s>>>(np, old[k]);
        if (!group) part_barrier(q, q->stream);  // nobody steps until every rank has pulled
    }
    if ((st = group ? group_sync(g) : fetch_ctl(g))) return st;
    if (cudaGetLastError() != cudaSuccess) return SWAMP_E_CUDA;
    for (swamp_gpu* q : mine) {
        cudaSetDevice(q->device);
        apply_bounds(q->P, nb);
        for (cudaGraphExec_t* e : {&q->graph1, &q->graphS})
            if (*e) {
                cudaGraphExecDestroy(*e);
                *e = nullptr;
            }
    }
    if (group && g->serial) {
        for (cudaGraphExec_t* e : {&g->graph1, &g->graphS})
            if (*e) {
                cudaGraphExecDestroy(*e);
                *e = nullptr;
            }
        cudaSetDevice(q0->device);
        if ((st = capture_step_graphs(g, q0->stream, [&] { serial_enqueue_step(g); }))) return st;
    } else {
        for (swamp_gpu* q : mine) {
            cudaSetDevice(q->device);
            if ((st = part_build_graphs(q))) return st;
        }
    }
    if (changed) *changed = 1;
    return group ? group_sync(g) : fetch_ctl(g);
}

#define SWAMP_STR2(x) #x
#define SWAMP_STR(x) SWAMP_STR2(x)
const char* swamp_gpu_build_info(void) {
    return "libswamp_gpu: sm_100a, --fmad=false, nvcc " SWAMP_STR(__CUDACC_VER_MAJOR__) "." SWAMP_STR(__CUDACC_VER_MINOR__);
}

}  // extern "C"
