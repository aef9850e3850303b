// c_api.cu -- the extern "C" boundary (include/adakv_b200.h): host-side validation
// mirroring the reference's throw sites, workspace carving, stream-ordered launches.
#include <cstdio>
#include <cstring>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "select.cuh"

namespace adakv_b200 {

// ---- defined in the kernel translation units
size_t score_window_generic_workspace(adakv_dtype dt, const adakv_layer_shape& s);
adakv_status score_window_generic(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel,
                                  int32_t scale, const void* q, const void* k, void* head_scores,
                                  void* group_scores, void* ws, uint32_t* err, cudaStream_t stream);
size_t score_window_generic_smem(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel);
bool score_window_tc_supported(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel);
size_t score_window_tc_workspace(const adakv_layer_shape& s);
adakv_status score_window_tc(const adakv_layer_shape& s, int64_t pool_kernel, int32_t scale,
                             const void* q, const void* k, void* head_scores, void* group_scores,
                             void* ws, uint32_t* err, cudaStream_t stream);


adakv_status launch_layout(const int32_t* budgets, int64_t P, int64_t G, int64_t m, int64_t reserve,
                           int64_t layer_budget, const int64_t* layer_budgets, int32_t* seg_start,
                           int32_t* seqlens, int32_t* seg_cap, cudaStream_t stream);
adakv_status launch_gather(adakv_dtype dt, const adakv_layer_shape& s, int64_t max_rows,
                           const void* k, const void* v, const int32_t* budgets,
                           const int32_t* kept_pos, int64_t kept_stride, const int32_t* seg_start,
                           void* k_cache, void* v_cache, uint32_t* err, cudaStream_t stream);
adakv_status launch_validate(adakv_dtype dt, const void* data, int64_t n, uint32_t* err, cudaStream_t stream);
size_t decode_workspace_bytes(int64_t P, int64_t H, int64_t G, int64_t d, int64_t max_rows, size_t acc);
adakv_status launch_decode(adakv_dtype dt, int64_t P, int64_t H, int64_t G, int64_t d, int32_t scale,
                           const void* q, void* kc, void* vc, int64_t cache_rows, const int32_t* ss,
                           const int32_t* cap, int32_t* sl, int64_t max_rows, const void* kn, const void* vn,
                           void* out, void* ws, uint32_t* err, bool overlap_prev, cudaStream_t stream);
adakv_status launch_append(adakv_dtype dt, int64_t segments, int64_t rows, int64_t d, void* kc, void* vc,
                           const int32_t* ss, const int32_t* cap, int32_t* sl, const void* kn, const void* vn,
                           uint32_t* err, cudaStream_t stream);
__global__ void budget_kernel(int op, const double* quotas_in, const int64_t* a_in, int64_t h,
                              int64_t total, double alpha, double bmax, double bmin,
                              const int64_t* caps_in, int64_t* out, double* quotas,
                              uint64_t* caps, uint64_t* tmp_a, uint64_t* tmp_o, uint32_t* err);

// ---------------------------------------------------------------- launch ordering
// The decode kernel reads its segments' rows, lengths and capacities before
// griddepcontrol.wait, so it overlaps (programmatic dependent launch) its predecessor only
// when the caller vouches, per call, that the predecessor writes none of them
// (ADAKV_DECODE_CHAINED: a decode of other segments).  adakv_set_decode_overlap(0) turns
// the overlap off globally (A/B measurements).
namespace {
std::atomic<int> g_decode_overlap{-1};
}  // namespace

static bool decode_overlap_enabled() {
    int v = g_decode_overlap.load();
    if (v < 0) {
        const char* e = std::getenv("ADAKV_DECODE_OVERLAP");
        v = (e && e[0] == '0') ? 0 : 1;
        g_decode_overlap.store(v);
    }
    return v != 0;
}

// ---------------------------------------------------------------- errors
namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
adakv_status fail(adakv_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}
adakv_status cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                   ") in " + what;
    return ADAKV_CUDA_ERROR;
}

int device_sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

namespace {

// config.validate(), policies.hpp:65-72
adakv_status validate_config(const adakv_policy_config* c) {
    if (!c) return fail(ADAKV_INVALID_ARGUMENT, "PolicyConfig: null");
    if (c->window_size < 1) return fail(ADAKV_INVALID_ARGUMENT, "PolicyConfig: window_size < 1");
    if (c->pool_kernel % 2 == 0 || c->pool_kernel <= 0)
        return fail(ADAKV_INVALID_ARGUMENT, "PolicyConfig: pool_kernel must be odd");
    if (!(c->alpha >= 0.0 && c->alpha <= 1.0))
        return fail(ADAKV_INVALID_ARGUMENT, "PolicyConfig: alpha outside [0,1]");
    if (c->gqa_group_size <= 0) return fail(ADAKV_INVALID_ARGUMENT, "PolicyConfig: zero group size");
    if (c->kind < ADAKV_SNAPKV || c->kind > ADAKV_STREAMING_LLM)
        return fail(ADAKV_INVALID_ARGUMENT, "unknown policy kind");
    return ADAKV_OK;
}

adakv_status validate_dtype(adakv_dtype dt) {
    if (dt != ADAKV_F32 && dt != ADAKV_F64 && dt != ADAKV_BF16)
        return fail(ADAKV_INVALID_ARGUMENT, "unknown dtype");
    return ADAKV_OK;
}

// window_scores / attention_weights preconditions (policies.hpp:121, attention.hpp:170-172)
adakv_status validate_shape(const adakv_layer_shape* s) {
    if (!s) return fail(ADAKV_INVALID_ARGUMENT, "shape: null");
    if (s->problems < 0) return fail(ADAKV_INVALID_ARGUMENT, "shape: negative problem count");
    if (s->kv_groups <= 0 || s->q_heads <= 0) return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: head count mismatch");
    if (s->q_heads % s->kv_groups != 0)
        return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: head count not divisible by group");
    if (s->window <= 0) return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: empty window");
    if (s->outside <= 0) return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: empty outside cache head");
    if (s->head_dim <= 0) return fail(ADAKV_INVALID_ARGUMENT, "attention_weights: head dim mismatch");
    if (s->kv_groups > kMaxSeg) return fail(ADAKV_UNSUPPORTED, "more than 64 KV groups per problem");
    return ADAKV_OK;
}

size_t acc_size(adakv_dtype dt) { return dt == ADAKV_F64 ? 8 : 4; }

std::atomic<int> g_tc_enabled{-1};  // -1: from ADAKV_DISABLE_TC at first use

bool use_tc(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel) {
    int en = g_tc_enabled.load();
    if (en < 0) {
        const char* e = std::getenv("ADAKV_DISABLE_TC");
        en = (e && e[0] == '1') ? 0 : 1;
        g_tc_enabled.store(en);
    }
    return en && score_window_tc_supported(dt, s, pool_kernel);
}

size_t score_ws(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel) {
    return use_tc(dt, s, pool_kernel) ? score_window_tc_workspace(s) : score_window_generic_workspace(dt, s);
}

adakv_status run_scores(adakv_dtype dt, const adakv_layer_shape& s, int64_t pool_kernel, int32_t scale,
                        const void* q, const void* k, void* hs, void* gs, void* ws, uint32_t* err, cudaStream_t st) {
    if (use_tc(dt, s, pool_kernel)) return score_window_tc(s, pool_kernel, scale, q, k, hs, gs, ws, err, st);
    const size_t smem = score_window_generic_smem(dt, s, pool_kernel);
    if (smem > 227 * 1024)
        return fail(ADAKV_UNSUPPORTED, "window_scores: shape exceeds the generic kernel's shared memory");
    return score_window_generic(dt, s, pool_kernel, scale, q, k, hs, gs, ws, err, st);
}

struct CompressLayout {
    uint32_t* err;
    void* scores;
    int32_t* kept_pos;
    int64_t kept_stride;
    int64_t* totals;
    void* score_ws;
    size_t bytes;
};

CompressLayout compress_layout(void* base, adakv_dtype dt, const adakv_layer_shape& s,
                               int64_t pool_kernel, bool own_scores, bool per_problem) {
    CompressLayout L{};
    Arena ar(base);
    L.err = ar.take<uint32_t>(kWsHeader / 4);
    const size_t n = size_t(s.problems * s.kv_groups * s.outside);
    L.scores = own_scores ? static_cast<void*>(ar.take<char>(n * acc_size(dt))) : nullptr;
    L.kept_stride = s.kv_groups * s.outside;
    L.kept_pos = ar.take<int32_t>(size_t(s.problems * L.kept_stride));
    L.totals = per_problem ? ar.take<int64_t>(size_t(s.problems)) : nullptr;
    L.score_ws = ar.take<char>(score_ws(dt, s, pool_kernel));
    L.bytes = ar.off + 256;
    return L;
}

// per-problem layer budgets outside the reference's floor / capacity (policies.hpp:229-231,
// budget.hpp:48-59) latch ERR_BUDGET and become a zero outside total; select then rejects
// the problem (zero budgets, nothing indexed)
__global__ void outside_totals_kernel(const int64_t* lb, int64_t P, int64_t m, int64_t G, int64_t n_o, int64_t* out,
                                      uint32_t* err) {
    for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += blockDim.x * gridDim.x) {
        const int64_t b = lb[i];
        const bool ok = b >= m * G + G && b - m * G <= G * n_o;
        out[i] = ok ? b - m * G : -1;
        if (!ok) atomicOr(err, ERR_BUDGET);
    }
}


adakv_status run_budget_kernel(int op, const double* quotas, const int64_t* a, int64_t h,
                               int64_t total, double alpha, double bmax, double bmin,
                               const int64_t* caps, int64_t* out, uint32_t* err_out) {
    const size_t n = size_t(h > 0 ? h : 1);
    char* dbuf = nullptr;
    const size_t bytes = n * (8 * 7) + 64;
    ADAKV_CUDA_TRY(cudaMalloc(&dbuf, bytes));
    double* d_qin = reinterpret_cast<double*>(dbuf);
    int64_t* d_a = reinterpret_cast<int64_t*>(d_qin + n);
    int64_t* d_caps = d_a + n;
    int64_t* d_out = d_caps + n;
    double* d_quotas = reinterpret_cast<double*>(d_out + n);
    uint64_t* d_capsu = reinterpret_cast<uint64_t*>(d_quotas + n);
    uint64_t* d_tmpa = d_capsu + n;
    uint32_t* d_err = reinterpret_cast<uint32_t*>(d_tmpa + n);
    uint64_t* d_tmpo = nullptr;
    cudaError_t e = cudaMalloc(&d_tmpo, n * 8);
    if (e == cudaSuccess && quotas) e = cudaMemcpy(d_qin, quotas, size_t(h) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && a) e = cudaMemcpy(d_a, a, size_t(h) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && caps) e = cudaMemcpy(d_caps, caps, size_t(h) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        budget_kernel<<<1, 32>>>(op, d_qin, d_a, h, total, alpha, bmax, bmin, caps ? d_caps : nullptr,
                                 d_out, d_quotas, d_capsu, d_tmpa, d_tmpo, d_err);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d_out, size_t(h) * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(err_out, d_err, 4, cudaMemcpyDeviceToHost);
    cudaFree(d_tmpo);
    cudaFree(dbuf);
    if (e != cudaSuccess) return cuda_fail(e, "budget kernel");
    return ADAKV_OK;
}

// host-side precondition of detail::apportion (budget.hpp:48-59)
adakv_status apportion_precheck(const double* quotas, int64_t h, int64_t total, const int64_t* caps) {
    uint64_t cap_sum = 0;
    for (int64_t i = 0; i < h; ++i) {
        const uint64_t c = caps ? uint64_t(caps[i]) : kAmpleCap;
        cap_sum = cap_sum > ~uint64_t(0) - c ? ~uint64_t(0) : cap_sum + c;
    }
    if (uint64_t(total) > cap_sum) return fail(ADAKV_INVALID_ARGUMENT, "apportion: total exceeds capacity");
    if (quotas)
        for (int64_t i = 0; i < h; ++i)
            if (!(quotas[i] >= 0.0)) return fail(ADAKV_INVALID_ARGUMENT, "apportion: negative quota");
    return ADAKV_OK;
}

}  // namespace
}  // namespace adakv_b200

using namespace adakv_b200;

extern "C" {

const char* adakv_last_error(void) { return g_last_error.c_str(); }
int adakv_abi_version(void) { return ADAKV_B200_ABI_VERSION; }

int adakv_set_tensor_core_scoring(int enabled) {
    const int prev = g_tc_enabled.exchange(enabled ? 1 : 0);
    return prev;
}

adakv_status adakv_workspace_status(const void* workspace, adakv_stream_t stream) {
    uint32_t e = 0;
    ADAKV_CUDA_TRY(cudaMemcpyAsync(&e, workspace, 4, cudaMemcpyDeviceToHost, stream));
    ADAKV_CUDA_TRY(cudaStreamSynchronize(stream));
    if (e & ERR_NONFINITE) return fail(ADAKV_INVALID_ARGUMENT, "LayerCache: non-finite entry");
    if (e & ERR_REPAIR) return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: cannot guarantee one element per head");
    if (e & ERR_BUDGET) return fail(ADAKV_INVALID_ARGUMENT, "topk_decision: k exceeds length");
    if (e & ERR_CAPACITY) return fail(ADAKV_INVALID_ARGUMENT, "append_kv: capacity exhausted");
    if (e & ERR_MAXROWS) return fail(ADAKV_INVALID_ARGUMENT, "decode: segment longer than max_rows");
    return ADAKV_OK;
}

adakv_status adakv_clear_workspace_status(void* workspace, adakv_stream_t stream) {
    if (!workspace) return fail(ADAKV_INVALID_ARGUMENT, "workspace: null");
    ADAKV_CUDA_TRY(cudaMemsetAsync(workspace, 0, 4, reinterpret_cast<cudaStream_t>(stream)));
    return ADAKV_OK;
}

adakv_status adakv_validate_finite(adakv_dtype dtype, const void* data, int64_t n, void* workspace,
                                   adakv_stream_t stream) {
    ADAKV_TRY(validate_dtype(dtype));
    if (n < 0) return fail(ADAKV_INVALID_ARGUMENT, "validate: negative element count");
    if (!workspace) return fail(ADAKV_INVALID_ARGUMENT, "validate: null workspace");
    if (n == 0) return ADAKV_OK;
    if (!data) return fail(ADAKV_INVALID_ARGUMENT, "validate: null data");
    return launch_validate(dtype, data, n, static_cast<uint32_t*>(workspace), reinterpret_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------------ scoring
adakv_status adakv_window_scores_workspace(adakv_dtype dtype, const adakv_layer_shape* shape,
                                           size_t* bytes) {
    ADAKV_TRY(validate_dtype(dtype));
    ADAKV_TRY(validate_shape(shape));
    *bytes = kWsHeader + 256 + score_ws(dtype, *shape, 7);
    return ADAKV_OK;
}

adakv_status adakv_window_scores(adakv_dtype dtype, const adakv_layer_shape* shape, int64_t pool_kernel,
                                 int32_t scale, const void* q, const void* k, void* head_scores,
                                 void* group_scores, void* workspace, size_t workspace_bytes,
                                 adakv_stream_t stream) {
    ADAKV_TRY(validate_dtype(dtype));
    ADAKV_TRY(validate_shape(shape));
    if (pool_kernel % 2 == 0 || pool_kernel <= 0)
        return fail(ADAKV_INVALID_ARGUMENT, "maxpool: kernel must be odd");
    const size_t need = kWsHeader + 256 + score_ws(dtype, *shape, pool_kernel);
    if (workspace_bytes < need) return fail(ADAKV_WORKSPACE_TOO_SMALL, "window_scores: workspace too small");
    if (shape->problems == 0) return ADAKV_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ADAKV_CUDA_TRY(cudaMemsetAsync(workspace, 0, 4, st));
    void* ws = static_cast<char*>(workspace) + kWsHeader;
    return run_scores(dtype, *shape, pool_kernel, scale, q, k, head_scores, group_scores, ws,
                      static_cast<uint32_t*>(workspace), st);
}

// ------------------------------------------------------------------ selection
adakv_status adakv_segmented_select_workspace(int64_t problems, int64_t segments, size_t* bytes) {
    (void)problems;
    (void)segments;
    *bytes = kWsHeader;
    return ADAKV_OK;
}

adakv_status adakv_segmented_select(adakv_dtype key_dtype, int64_t problems, int64_t segments,
                                    const int64_t* seg_off, const void* scores, int64_t total,
                                    const int64_t* totals, const adakv_select_config* cfg,
                                    int32_t* raw_counts, int32_t* budgets, uint8_t* keep,
                                    int32_t* kept_pos, int64_t kept_stride, void* workspace,
                                    size_t workspace_bytes, adakv_stream_t stream) {
    if (key_dtype != ADAKV_F32 && key_dtype != ADAKV_F64)
        return fail(ADAKV_INVALID_ARGUMENT, "segmented_select: keys must be f32 or f64");
    if (segments <= 0) return fail(ADAKV_INVALID_ARGUMENT, "adaptive_allocation: no heads");
    if (segments > kMaxSeg) return fail(ADAKV_UNSUPPORTED, "segmented_select: more than 64 segments");
    if (!cfg || !budgets) return fail(ADAKV_INVALID_ARGUMENT, "segmented_select: null argument");
    if (workspace_bytes < kWsHeader) return fail(ADAKV_WORKSPACE_TOO_SMALL, "segmented_select: workspace too small");
    SelParams prm{};
    if (seg_off[0] != 0) return fail(ADAKV_INVALID_ARGUMENT, "segmented_select: seg_off[0] != 0");
    for (int64_t s = 0; s <= segments; ++s) {
        prm.off[s] = seg_off[s];
        if (s && seg_off[s] < seg_off[s - 1]) return fail(ADAKV_INVALID_ARGUMENT, "segmented_select: offsets decrease");
    }
    const int64_t N = seg_off[segments];
    if (cfg->alloc_mode == ADAKV_ALLOC_ADAPTIVE && !totals && total > N)
        return fail(ADAKV_INVALID_ARGUMENT, "adaptive_allocation: total exceeds element count");
    if (cfg->alloc_mode == ADAKV_ALLOC_UNIFORM && !totals && total > N)
        return fail(ADAKV_INVALID_ARGUMENT, "apportion: total exceeds capacity");
    if (cfg->blend && !(cfg->alpha >= 0.0 && cfg->alpha <= 1.0))
        return fail(ADAKV_INVALID_ARGUMENT, "safeguard_blend: alpha outside [0,1]");
    if (total < 0) return fail(ADAKV_INVALID_ARGUMENT, "segmented_select: negative total");
    if (kept_pos && kept_stride < (cfg->alloc_mode == ADAKV_ALLOC_GIVEN ? N : (totals ? N : total)))
        return fail(ADAKV_INVALID_ARGUMENT, "segmented_select: kept_stride too small");
    if (problems == 0) return ADAKV_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ADAKV_CUDA_TRY(cudaMemsetAsync(workspace, 0, 4, st));
    prm.S = int(segments);
    prm.N = N;
    prm.alloc_mode = cfg->alloc_mode;
    prm.blend = cfg->blend;
    prm.repair = cfg->repair;
    prm.streaming = cfg->streaming;
    prm.alpha = cfg->alpha;
    prm.sink = cfg->sink_tokens;
    prm.total = total;
    prm.totals = totals;
    prm.scores = scores;
    prm.raw_counts = raw_counts;
    prm.budgets = budgets;
    prm.keep = keep;
    prm.kept_pos = kept_pos;
    prm.kept_stride = kept_stride;
    prm.err = static_cast<uint32_t*>(workspace);
    return launch_select(key_dtype == ADAKV_F64, problems, prm, st);
}

// ------------------------------------------------------------------ gather
adakv_status adakv_gather(adakv_dtype dtype, const adakv_layer_shape* shape, int64_t layer_budget,
                          const int64_t* layer_budgets, const void* k, const void* v, const int32_t* budgets,
                          const int32_t* kept_pos, int64_t kept_stride, int64_t reserve, void* k_cache,
                          void* v_cache, int32_t* seg_start, int32_t* seqlens, int32_t* seg_cap, void* workspace,
                          adakv_stream_t stream) {
    ADAKV_TRY(validate_dtype(dtype));
    ADAKV_TRY(validate_shape(shape));
    if (reserve < 0) return fail(ADAKV_INVALID_ARGUMENT, "gather: negative reserve");
    if (shape->problems == 0) return ADAKV_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t G = shape->kv_groups, m = shape->window;
    ADAKV_TRY(launch_layout(budgets, shape->problems, G, m, reserve, layer_budget, layer_budgets, seg_start,
                            seqlens, seg_cap, st));
    const int64_t max_rows = layer_budgets ? G * (shape->outside + m) : layer_budget;
    return launch_gather(dtype, *shape, max_rows, k, v, budgets, kept_pos, kept_stride, seg_start, k_cache,
                         v_cache, static_cast<uint32_t*>(workspace), st);
}

// ------------------------------------------------------------------ compress
int64_t adakv_cache_rows(const adakv_layer_shape* shape, int64_t layer_budget,
                         const int64_t* layer_budgets_host, int64_t reserve) {
    if (!shape) return -1;
    int64_t rows = 0;
    for (int64_t p = 0; p < shape->problems; ++p)
        rows += (layer_budgets_host ? layer_budgets_host[p] : layer_budget) + shape->kv_groups * reserve;
    return rows;
}

adakv_status adakv_compress_workspace(adakv_dtype dtype, const adakv_layer_shape* shape,
                                      const adakv_policy_config* cfg, size_t* bytes) {
    ADAKV_TRY(validate_dtype(dtype));
    ADAKV_TRY(validate_shape(shape));
    ADAKV_TRY(validate_config(cfg));
    *bytes = compress_layout(nullptr, dtype, *shape, cfg->pool_kernel, true, true).bytes;
    return ADAKV_OK;
}

static adakv_status compress_impl(adakv_dtype dtype, const adakv_layer_shape* shape, const adakv_policy_config* cfg,
                                  int64_t layer_budget, const int64_t* layer_budgets, const void* q, const void* k,
                                  const void* v, int64_t reserve, void* k_cache, void* v_cache, int32_t* seg_start,
                                  int32_t* seqlens, int32_t* seg_cap, int32_t* budgets, void* group_scores,
                                  uint8_t* keep, void* workspace, size_t workspace_bytes, adakv_stream_t stream,
                                  adakv_stream_t gather_stream) {
    ADAKV_TRY(validate_dtype(dtype));
    ADAKV_TRY(validate_config(cfg));
    ADAKV_TRY(validate_shape(shape));
    const adakv_layer_shape& s = *shape;
    const int64_t G = s.kv_groups, m = s.window, n_o = s.outside;
    if (s.q_heads / G != cfg->gqa_group_size)
        return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: head count mismatch");
    if (!budgets || !seg_start || !seqlens || !k_cache || !v_cache)
        return fail(ADAKV_INVALID_ARGUMENT, "compress: null output");
    if (reserve < 0) return fail(ADAKV_INVALID_ARGUMENT, "compress: negative reserve");
    if (!layer_budgets) {
        // policies.hpp:229-231 and the capacity checks of apportion / adaptive_allocation
        if (layer_budget < m * G + G)
            return fail(ADAKV_INVALID_ARGUMENT, "evict_layer: budget below the window-plus-one floor");
        if (layer_budget - m * G > G * n_o)
            return fail(ADAKV_INVALID_ARGUMENT, "apportion: total exceeds capacity");
    }
    const CompressLayout L = compress_layout(workspace, dtype, s, cfg->pool_kernel, group_scores == nullptr,
                                             layer_budgets != nullptr);
    if (workspace_bytes < L.bytes) return fail(ADAKV_WORKSPACE_TOO_SMALL, "compress: workspace too small");
    if (s.problems == 0) return ADAKV_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ADAKV_CUDA_TRY(cudaMemsetAsync(workspace, 0, 4, st));
    void* scores = group_scores ? group_scores : L.scores;

    // K1: observation-window scores for every group (scoring runs for every kind,
    // policies.hpp:239-247)
    ADAKV_TRY(run_scores(dtype, s, cfg->pool_kernel, cfg->scale, q, k, nullptr, scores, L.score_ws, L.err, st));

    // K2/K3 selection
    SelParams prm{};
    for (int64_t g = 0; g <= G; ++g) prm.off[g] = g * n_o;
    prm.S = int(G);
    prm.N = G * n_o;
    const bool ada = cfg->kind == ADAKV_ADA_SNAPKV || cfg->kind == ADAKV_ADA_PYRAMID;
    prm.alloc_mode = ada ? ADAKV_ALLOC_ADAPTIVE : ADAKV_ALLOC_UNIFORM;
    prm.blend = ada ? 1 : 0;
    prm.repair = 1;
    prm.streaming = cfg->kind == ADAKV_STREAMING_LLM;
    prm.alpha = cfg->alpha;
    prm.sink = cfg->sink_tokens;
    prm.total = layer_budget - m * G;
    if (layer_budgets) {
        outside_totals_kernel<<<unsigned(ceil_div(s.problems, 256)), 256, 0, st>>>(layer_budgets, s.problems, m,
                                                                                G, n_o, L.totals, L.err);
        ADAKV_CUDA_TRY(cudaGetLastError());
        prm.totals = L.totals;
    }
    prm.scores = scores;
    prm.nonneg = 1;  // window scores: means of softmax probabilities, +0 or positive
    prm.budgets = budgets;
    prm.keep = keep;
    prm.kept_pos = L.kept_pos;
    prm.kept_stride = L.kept_stride;
    prm.err = L.err;
    ADAKV_TRY(launch_select(dtype == ADAKV_F64, s.problems, prm, st));

    // layout + K3 gather into the varlen planes
    ADAKV_TRY(launch_layout(budgets, s.problems, G, m, reserve, layer_budget, layer_budgets, seg_start,
                            seqlens, seg_cap, st));
    const int64_t max_rows = layer_budgets ? G * (n_o + m) : layer_budget;
    cudaStream_t gst = st;
    if (gather_stream && reinterpret_cast<cudaStream_t>(gather_stream) != st) {
        // fork: the gather waits for the layout on `stream`, which itself goes on
        gst = reinterpret_cast<cudaStream_t>(gather_stream);
        cudaEvent_t ev;
        ADAKV_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        cudaError_t e = cudaEventRecord(ev, st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(gst, ev, 0);
        cudaEventDestroy(ev);  // released once the wait has been satisfied
        ADAKV_CUDA_TRY(e);
    }
    return launch_gather(dtype, s, max_rows, k, v, budgets, L.kept_pos, L.kept_stride, seg_start, k_cache,
                         v_cache, L.err, gst);
}

adakv_status adakv_compress(adakv_dtype dtype, const adakv_layer_shape* shape, const adakv_policy_config* cfg,
                            int64_t layer_budget, const int64_t* layer_budgets, const void* q,
                            const void* k, const void* v, int64_t reserve, void* k_cache, void* v_cache,
                            int32_t* seg_start, int32_t* seqlens, int32_t* seg_cap, int32_t* budgets,
                            void* group_scores,
                            uint8_t* keep, void* workspace, size_t workspace_bytes, adakv_stream_t stream) {
    return compress_impl(dtype, shape, cfg, layer_budget, layer_budgets, q, k, v, reserve, k_cache, v_cache, seg_start,
                         seqlens, seg_cap, budgets, group_scores, keep, workspace, workspace_bytes, stream, nullptr);
}

adakv_status adakv_compress_split(adakv_dtype dtype, const adakv_layer_shape* shape, const adakv_policy_config* cfg,
                                  int64_t layer_budget, const int64_t* layer_budgets, const void* q, const void* k,
                                  const void* v, int64_t reserve, void* k_cache, void* v_cache, int32_t* seg_start,
                                  int32_t* seqlens, int32_t* seg_cap, int32_t* budgets, void* group_scores,
                                  uint8_t* keep, void* workspace, size_t workspace_bytes, adakv_stream_t stream,
                                  adakv_stream_t gather_stream) {
    return compress_impl(dtype, shape, cfg, layer_budget, layer_budgets, q, k, v, reserve, k_cache, v_cache, seg_start,
                         seqlens, seg_cap, budgets, group_scores, keep, workspace, workspace_bytes, stream,
                         gather_stream);
}

// ------------------------------------------------------------------ decode
adakv_status adakv_decode_workspace(int64_t problems, int64_t q_heads, int64_t kv_groups, int64_t head_dim,
                                    int64_t max_rows, size_t* bytes) {
    *bytes = kWsHeader + decode_workspace_bytes(problems, q_heads, kv_groups, head_dim, max_rows, 8);
    return ADAKV_OK;
}

adakv_status adakv_decode(adakv_dtype dtype, int64_t problems, int64_t q_heads, int64_t kv_groups,
                          int64_t head_dim, int32_t scale, const void* q, void* k_cache, void* v_cache,
                          int64_t cache_rows, const int32_t* seg_start, const int32_t* seg_cap, int32_t* seqlens,
                          int64_t max_rows, const void* k_new, const void* v_new, void* out, void* workspace,
                          size_t workspace_bytes, uint32_t flags, adakv_stream_t stream) {
    ADAKV_TRY(validate_dtype(dtype));
    if (kv_groups <= 0 || q_heads <= 0 || q_heads % kv_groups != 0)
        return fail(ADAKV_INVALID_ARGUMENT, "attention_output: head count mismatch");
    if (head_dim <= 0) return fail(ADAKV_INVALID_ARGUMENT, "attention_weights: head dim mismatch");
    if ((k_new == nullptr) != (v_new == nullptr))
        return fail(ADAKV_INVALID_ARGUMENT, "append_kv: k and v must both be given");
    if (max_rows <= 0) return fail(ADAKV_INVALID_ARGUMENT, "attention_weights: empty key set");
    if (cache_rows <= 0) return fail(ADAKV_INVALID_ARGUMENT, "decode: empty cache plane");
    if (!seg_start || !seqlens || !seg_cap) return fail(ADAKV_INVALID_ARGUMENT, "decode: null segment table");
    if (flags & ~uint32_t(ADAKV_DECODE_CHAINED)) return fail(ADAKV_INVALID_ARGUMENT, "decode: unknown flags");
    const size_t need = kWsHeader + decode_workspace_bytes(problems, q_heads, kv_groups, head_dim, max_rows,
                                                           acc_size(dtype));
    if (workspace_bytes < need) return fail(ADAKV_WORKSPACE_TOO_SMALL, "decode: workspace too small");
    if (problems == 0) return ADAKV_OK;
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const bool overlap = (flags & ADAKV_DECODE_CHAINED) && decode_overlap_enabled();
    return launch_decode(dtype, problems, q_heads, kv_groups, head_dim, scale, q, k_cache, v_cache, cache_rows,
                         seg_start, seg_cap, seqlens, max_rows, k_new, v_new, out,
                         static_cast<char*>(workspace) + kWsHeader, static_cast<uint32_t*>(workspace), overlap, st);
}

adakv_status adakv_host_device_pointer(const void* host, void** device_ptr) {
    if (!host || !device_ptr) return fail(ADAKV_INVALID_ARGUMENT, "host_device_pointer: null argument");
    cudaPointerAttributes at{};
    const cudaError_t e = cudaPointerGetAttributes(&at, host);
    if (e != cudaSuccess || at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) {
        cudaGetLastError();
        return fail(ADAKV_INVALID_ARGUMENT, "host_device_pointer: not pinned host memory mapped into the device");
    }
    *device_ptr = at.devicePointer;
    return ADAKV_OK;
}

int adakv_set_decode_overlap(int enabled) {
    const int prev = decode_overlap_enabled() ? 1 : 0;
    g_decode_overlap.store(enabled ? 1 : 0);
    return prev;
}

adakv_status adakv_append_rows(adakv_dtype dtype, int64_t segments, int64_t rows, int64_t head_dim,
                               void* k_cache, void* v_cache, const int32_t* seg_start, const int32_t* seg_cap,
                               int32_t* seqlens, const void* k_new, const void* v_new, void* workspace,
                               adakv_stream_t stream) {
    ADAKV_TRY(validate_dtype(dtype));
    if (segments < 0) return fail(ADAKV_OUT_OF_RANGE, "append_kv: head index out of range");
    if (rows < 0) return fail(ADAKV_INVALID_ARGUMENT, "append_kv: negative row count");
    if (segments == 0 || rows == 0) return ADAKV_OK;
    if (k_new == nullptr || v_new == nullptr) return fail(ADAKV_INVALID_ARGUMENT, "append_kv: k and v must both be given");
    if (!seg_start || !seg_cap || !seqlens) return fail(ADAKV_INVALID_ARGUMENT, "append_kv: null segment table");
    if (!workspace) return fail(ADAKV_INVALID_ARGUMENT, "append_kv: null workspace");
    return launch_append(dtype, segments, rows, head_dim, k_cache, v_cache, seg_start, seg_cap, seqlens, k_new,
                         v_new, static_cast<uint32_t*>(workspace), reinterpret_cast<cudaStream_t>(stream));
}

adakv_status adakv_append_kv(adakv_dtype dtype, int64_t segments, int64_t head_dim, void* k_cache,
                             void* v_cache, const int32_t* seg_start, const int32_t* seg_cap, int32_t* seqlens,
                             const void* k_new, const void* v_new, void* workspace, adakv_stream_t stream) {
    return adakv_append_rows(dtype, segments, 1, head_dim, k_cache, v_cache, seg_start, seg_cap, seqlens, k_new,
                             v_new, workspace, stream);
}

// ------------------------------------------------------------------ budget helpers
adakv_status adakv_apportion(const double* quotas, int64_t h, int64_t total, const int64_t* caps,
                             int64_t* out) {
    ADAKV_TRY(apportion_precheck(quotas, h, total, caps));
    if (h == 0) return ADAKV_OK;
    uint32_t e = 0;
    ADAKV_TRY(run_budget_kernel(0, quotas, nullptr, h, total, 0, 0, 0, caps, out, &e));
    return e ? fail(ADAKV_INVALID_ARGUMENT, "apportion: failed") : ADAKV_OK;
}

adakv_status adakv_uniform_allocation(int64_t total, int64_t h, const int64_t* caps, int64_t* out) {
    if (h <= 0) return fail(ADAKV_INVALID_ARGUMENT, "uniform_allocation: no heads");
    ADAKV_TRY(apportion_precheck(nullptr, h, total, caps));
    uint32_t e = 0;
    ADAKV_TRY(run_budget_kernel(1, nullptr, nullptr, h, total, 0, 0, 0, caps, out, &e));
    return e ? fail(ADAKV_INVALID_ARGUMENT, "apportion: failed") : ADAKV_OK;
}

adakv_status adakv_safeguard_blend(const int64_t* adaptive, int64_t adaptive_total, int64_t total, int64_t h,
                                   double alpha, const int64_t* caps, int64_t* out) {
    if (adaptive_total != total) return fail(ADAKV_INVALID_ARGUMENT, "safeguard_blend: total mismatch");
    if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(ADAKV_INVALID_ARGUMENT, "safeguard_blend: alpha outside [0,1]");
    if (h <= 0) return fail(ADAKV_INVALID_ARGUMENT, "safeguard_blend: head count mismatch");
    ADAKV_TRY(apportion_precheck(nullptr, h, total, caps));
    uint32_t e = 0;
    ADAKV_TRY(run_budget_kernel(2, nullptr, adaptive, h, total, alpha, 0, 0, caps, out, &e));
    return e ? fail(ADAKV_INVALID_ARGUMENT, "apportion: failed") : ADAKV_OK;
}

adakv_status adakv_repair_zero_budgets(int64_t* counts, const int64_t* caps, int64_t h) {
    if (h <= 0) return ADAKV_OK;
    uint32_t e = 0;
    ADAKV_TRY(run_budget_kernel(3, nullptr, counts, h, 0, 0, 0, 0, caps, counts, &e));
    return e ? fail(ADAKV_INVALID_ARGUMENT, "evict_layer: cannot guarantee one element per head") : ADAKV_OK;
}

adakv_status adakv_pyramid_layer_budgets(int64_t per_layer_avg, int64_t num_layers, double beta_max,
                                         double beta_min, int64_t* out) {
    if (num_layers <= 0) return fail(ADAKV_INVALID_ARGUMENT, "pyramid_layer_budgets: zero layers");
    if (!(beta_min > 0.0) || beta_max < beta_min)
        return fail(ADAKV_INVALID_ARGUMENT, "pyramid_layer_budgets: invalid betas");
    uint32_t e = 0;
    ADAKV_TRY(run_budget_kernel(4, nullptr, nullptr, num_layers, per_layer_avg, 0, beta_max, beta_min, nullptr,
                                out, &e));
    return e ? fail(ADAKV_INVALID_ARGUMENT, "apportion: failed") : ADAKV_OK;
}

adakv_status adakv_device_malloc(void** ptr, size_t bytes) {
    ADAKV_CUDA_TRY(cudaMalloc(ptr, bytes > 0 ? bytes : 1));
    return ADAKV_OK;
}
adakv_status adakv_device_free(void* ptr) {
    ADAKV_CUDA_TRY(cudaFree(ptr));
    return ADAKV_OK;
}
adakv_status adakv_memcpy_to_device(void* dst, const void* src, size_t bytes) {
    if (bytes) ADAKV_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return ADAKV_OK;
}
adakv_status adakv_memcpy_to_host(void* dst, const void* src, size_t bytes) {
    if (bytes) ADAKV_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return ADAKV_OK;
}
adakv_status adakv_device_synchronize(void) {
    ADAKV_CUDA_TRY(cudaDeviceSynchronize());
    return ADAKV_OK;
}

}  // extern "C"
