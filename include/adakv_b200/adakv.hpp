// adakv.hpp -- C++ drop-in for the reference's hot-path API (namespace adakv, proj/include/adakv/),
// running on the B200 through the C ABI (include/adakv_b200.h).
//
// A reference user switches with
//     #include "adakv_b200/adakv.hpp"
//     namespace adakv = adakv_b200;
// and keeps calling window_scores / adaptive_allocation / safeguard_blend / topk_decision /
// evict_layer / evict_rows / attention_weights / attention_output / select_and_compact with the
// reference's exact signatures, value semantics and exception types.  Host doubles are marshalled
// to the device fp64 path (ADAKV_F64): budgets, decisions and compacted rows are the reference's
// bit for bit; scores and attention outputs agree to ~1e-15 relative (exp() ulps and the order of
// the softmax denominator sum).  Performance callers use the C ABI directly with bf16 planes.
//
// Scope: the compress + decode path.  The theory helpers (masked/renormalised
// weights, eviction loss), trace generator and report harness are not part of it.
// Deviations, all rejected with std::invalid_argument before any work: within a KV group every
// member head must hold identical K/V (the device stores each group once; the reference copies
// member rows, policies.hpp:276), and all groups must share one outside length (one n_o per call).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <initializer_list>
#include <istream>
#include <limits>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "adakv_b200.h"

namespace adakv_b200 {

/// Malformed or unsupported on-disk content (serde.hpp:18-21).
class FormatError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
/// Underlying I/O failure (serde.hpp:24-27).
class IoError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

namespace dev {

inline void check(adakv_status st) {
    if (st == ADAKV_OK) return;
    const std::string msg = adakv_last_error();
    switch (st) {
        case ADAKV_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case ADAKV_OUT_OF_RANGE: throw std::out_of_range(msg);
        case ADAKV_FORMAT_ERROR: throw FormatError(msg);
        case ADAKV_IO_ERROR: throw IoError(msg);
        default: throw std::runtime_error("adakv_b200: " + msg);
    }
}

/// Owning device buffer of T.
template <class T>
class Buffer {
  public:
    Buffer() = default;
    explicit Buffer(std::size_t n) : n_(n) { check(adakv_device_malloc(reinterpret_cast<void**>(&p_), bytes())); }
    Buffer(const T* host, std::size_t n) : Buffer(n) { upload(host, n); }
    Buffer(const Buffer&) = delete;
    Buffer& operator=(const Buffer&) = delete;
    ~Buffer() {
        if (p_) adakv_device_free(p_);
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }
    std::size_t bytes() const { return n_ * sizeof(T); }
    void upload(const T* host, std::size_t n) { check(adakv_memcpy_to_device(p_, host, n * sizeof(T))); }
    std::vector<T> download(std::size_t n) const {
        std::vector<T> out(n);
        check(adakv_memcpy_to_host(out.data(), p_, n * sizeof(T)));
        return out;
    }

  private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

inline std::vector<int64_t> to_i64(std::span<const std::size_t> v) {
    std::vector<int64_t> o(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) o[i] = int64_t(v[i]);
    return o;
}
inline std::vector<std::size_t> to_size(const std::vector<int64_t>& v) {
    std::vector<std::size_t> o(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) o[i] = std::size_t(v[i]);
    return o;
}
inline std::vector<std::size_t> to_size(const std::vector<int32_t>& v) {
    std::vector<std::size_t> o(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) o[i] = std::size_t(v[i]);
    return o;
}

}  // namespace dev

// --------------------------------------------------------------------------- L0 types
/// Dense row-major matrix of doubles (API of matrix.hpp:16-68).
class Matrix {
  public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0) : r_(rows), c_(cols), v_(rows * cols, fill) {}
    static Matrix from_rows(std::initializer_list<std::initializer_list<double>> rows) {
        Matrix m;
        for (const auto& row : rows) {
            if (m.r_ == 0) m.c_ = row.size();
            else if (row.size() != m.c_) throw std::invalid_argument("Matrix::from_rows: ragged rows");
            m.v_.insert(m.v_.end(), row.begin(), row.end());
            ++m.r_;
        }
        return m;
    }
    static Matrix identity(std::size_t n) {
        Matrix m(n, n);
        for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    bool empty() const { return v_.empty(); }
    double& operator()(std::size_t r, std::size_t c) { return v_[r * c_ + c]; }
    double operator()(std::size_t r, std::size_t c) const { return v_[r * c_ + c]; }
    std::span<double> row(std::size_t r) { return {v_.data() + r * c_, c_}; }
    std::span<const double> row(std::size_t r) const { return {v_.data() + r * c_, c_}; }
    std::span<const double> values() const { return v_; }
    std::span<double> values() { return v_; }
    void append_row(std::span<const double> row) {
        if (r_ == 0 && c_ == 0) c_ = row.size();
        if (row.size() != c_) throw std::invalid_argument("Matrix::append_row: width mismatch");
        v_.insert(v_.end(), row.begin(), row.end());
        ++r_;
    }
    bool operator==(const Matrix& o) const = default;

  private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<double> v_;
};

inline bool all_finite(std::span<const double> xs) {
    return std::all_of(xs.begin(), xs.end(), [](double x) { return std::isfinite(x); });
}
inline bool all_finite(const Matrix& m) { return all_finite(m.values()); }

/// matmul (matrix.hpp:91-102) on the device, same accumulation order.
inline Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimension mismatch");
    Matrix out(a.rows(), b.cols());
    if (a.rows() == 0 || b.cols() == 0) return out;
    if (a.cols() == 0) return out;
    dev::Buffer<double> da(a.values().data(), a.values().size()), db(b.values().data(), b.values().size());
    dev::Buffer<double> dq(out.values().size());
    dev::check(adakv_project_queries_f64(da.get(), db.get(), 1, int64_t(a.rows()), int64_t(a.cols()),
                                         int64_t(b.cols()), dq.get(), nullptr));
    const auto h = dq.download(out.values().size());
    std::copy(h.begin(), h.end(), out.values().begin());
    return out;
}

/// row_times (matrix.hpp:79-89): x (1 x r) times m (r x c), on the device.
inline std::vector<double> row_times(std::span<const double> x, const Matrix& m) {
    if (x.size() != m.rows()) throw std::invalid_argument("row_times: width mismatch");
    Matrix xm(1, x.size());
    std::copy(x.begin(), x.end(), xm.values().begin());
    const Matrix r = m.rows() ? matmul(xm, m) : Matrix(1, m.cols());
    return {r.values().begin(), r.values().end()};
}

// --------------------------------------------------------------------------- L1 types (attention.hpp:18-109)
struct HeadParams {
    Matrix wq, wk, wv, wo;
    std::size_t embed_dim() const { return wq.rows(); }
    std::size_t head_dim() const { return wq.cols(); }
    void validate() const {
        if (wk.rows() != wq.rows() || wv.rows() != wq.rows())
            throw std::invalid_argument("HeadParams: wq/wk/wv must share the embedding dim");
        if (wk.cols() != wq.cols() || wv.cols() != wq.cols() || wo.rows() != wq.cols())
            throw std::invalid_argument("HeadParams: projections must share the head dim");
        if (wo.cols() != wq.rows()) throw std::invalid_argument("HeadParams: wo must map back to the embedding dim");
        if (!all_finite(wq) || !all_finite(wk) || !all_finite(wv) || !all_finite(wo))
            throw std::invalid_argument("HeadParams: non-finite entry");
    }
};

struct LayerParams {
    std::vector<HeadParams> heads;
    std::size_t head_count() const { return heads.size(); }
    std::size_t embed_dim() const { return heads.front().embed_dim(); }
    std::size_t head_dim() const { return heads.front().head_dim(); }
    void validate() const {
        if (heads.empty()) throw std::invalid_argument("LayerParams: needs at least one head");
        for (const auto& h : heads) {
            h.validate();
            if (h.embed_dim() != embed_dim() || h.head_dim() != head_dim())
                throw std::invalid_argument("LayerParams: heads must share d and d_h");
        }
    }
};

struct HeadKV {
    Matrix keys, values;
    std::size_t length() const { return keys.rows(); }
};

struct LayerCache {
    std::vector<HeadKV> heads;
    std::size_t head_count() const { return heads.size(); }
    std::size_t total_elements() const {
        std::size_t n = 0;
        for (const auto& h : heads) n += h.length();
        return n;
    }
    void validate() const {
        for (const auto& h : heads) {
            if (h.keys.rows() != h.values.rows() || h.keys.cols() != h.values.cols())
                throw std::invalid_argument("LayerCache: keys/values shape mismatch");
            if (!all_finite(h.keys) || !all_finite(h.values)) throw std::invalid_argument("LayerCache: non-finite entry");
        }
    }
};

using WeightRow = std::vector<double>;
using WeightRows = std::vector<WeightRow>;
using AttentionWeights = std::vector<Matrix>;

struct EvictionDecision {
    std::vector<std::vector<std::uint8_t>> retain;
    std::size_t head_count() const { return retain.size(); }
    std::size_t retained_count(std::size_t i) const {
        return std::size_t(std::count_if(retain[i].begin(), retain[i].end(), [](std::uint8_t b) { return b != 0; }));
    }
    std::size_t total_retained() const {
        std::size_t c = 0;
        for (std::size_t i = 0; i < retain.size(); ++i) c += retained_count(i);
        return c;
    }
};

/// append_kv (attention.hpp:126-134): host-container append on the reference-typed cache
/// (the device cache appends inside adakv_decode / adakv_append_kv).
inline void append_kv(LayerCache& cache, std::size_t head, std::span<const double> k, std::span<const double> v) {
    if (head >= cache.heads.size()) throw std::out_of_range("append_kv: head index out of range");
    auto& slot = cache.heads[head];
    if (!slot.keys.empty() && (k.size() != slot.keys.cols() || v.size() != slot.values.cols()))
        throw std::invalid_argument("append_kv: row width mismatch");
    slot.keys.append_row(k);
    slot.values.append_row(v);
}

/// attention_weights (attention.hpp:169-179) on the device.
inline Matrix attention_weights(const Matrix& queries, const Matrix& keys, bool scale = true) {
    if (keys.rows() == 0) throw std::invalid_argument("attention_weights: empty key set");
    if (queries.cols() != keys.cols()) throw std::invalid_argument("attention_weights: head dim mismatch");
    Matrix w(queries.rows(), keys.rows());
    if (queries.rows() == 0) return w;
    dev::Buffer<double> dq(queries.values().data(), queries.values().size());
    dev::Buffer<double> dk(keys.values().data(), keys.values().size());
    dev::Buffer<double> dw(w.values().size());
    dev::check(adakv_attention_weights_f64(dq.get(), int64_t(queries.rows()), dk.get(), int64_t(keys.rows()),
                                           int64_t(keys.cols()), scale ? 1 : 0, dw.get(), nullptr));
    const auto h = dw.download(w.values().size());
    std::copy(h.begin(), h.end(), w.values().begin());
    return w;
}

/// attention_output (attention.hpp:182-196) on the device: y = sum_i A_i V_i W_i^O.
inline std::vector<double> attention_output(const WeightRows& weights, const LayerCache& cache,
                                            const LayerParams& params) {
    const std::size_t h = params.head_count();
    if (weights.size() != h || cache.head_count() != h)
        throw std::invalid_argument("attention_output: head count mismatch");
    std::vector<int64_t> woff(h + 1, 0), voff(h + 1, 0);
    for (std::size_t i = 0; i < h; ++i) {
        if (weights[i].size() != cache.heads[i].length())
            throw std::invalid_argument("attention_output: weight width mismatch");
        woff[i + 1] = woff[i] + int64_t(weights[i].size());
        voff[i + 1] = voff[i] + int64_t(cache.heads[i].length());
    }
    const std::size_t dh = params.head_dim(), D = params.embed_dim();
    std::vector<double> w, v, wo;
    for (std::size_t i = 0; i < h; ++i) {
        w.insert(w.end(), weights[i].begin(), weights[i].end());
        const auto vv = cache.heads[i].values.values();
        v.insert(v.end(), vv.begin(), vv.end());
        const auto ww = params.heads[i].wo.values();
        wo.insert(wo.end(), ww.begin(), ww.end());
    }
    dev::Buffer<double> dw(w.data(), std::max<std::size_t>(w.size(), 1)), dv(v.data(), std::max<std::size_t>(v.size(), 1));
    dev::Buffer<double> dwo(wo.data(), wo.size()), dctx(h * dh), dy(D);
    dev::Buffer<int64_t> dwoff(woff.data(), woff.size()), dvoff(voff.data(), voff.size());
    dev::check(adakv_attention_output_f64(dw.get(), dwoff.get(), dv.get(), dvoff.get(), int64_t(h), int64_t(dh),
                                          dwo.get(), int64_t(D), dctx.get(), dy.get(), nullptr));
    return dy.download(D);
}

// --------------------------------------------------------------------------- L2 budgets (budget.hpp)
enum class TieBreak { by_head_then_position };

struct BudgetAllocation {
    std::vector<std::size_t> per_head;
    std::size_t total = 0;
    std::size_t head_count() const { return per_head.size(); }
};

struct AllocationConfig {
    double alpha = 0.2;
    TieBreak tie_break = TieBreak::by_head_then_position;
};

namespace detail {

inline std::vector<std::size_t> ample_caps(std::size_t h) {
    return std::vector<std::size_t>(h, std::numeric_limits<std::size_t>::max() / 2);
}

/// detail::apportion (budget.hpp:45-93) on the device (bit-exact fp64).
inline std::vector<std::size_t> apportion(const std::vector<double>& quotas, std::size_t total,
                                          std::span<const std::size_t> caps) {
    if (caps.size() != quotas.size()) throw std::invalid_argument("apportion: caps length mismatch");
    std::vector<int64_t> out(quotas.size());
    const auto c = dev::to_i64(caps);
    dev::check(adakv_apportion(quotas.data(), int64_t(quotas.size()), int64_t(total), c.data(), out.data()));
    return dev::to_size(out);
}

/// detail::repair_zero_budgets (policies.hpp:178-196) on the device.
inline void repair_zero_budgets(std::vector<std::size_t>& counts, std::span<const std::size_t> caps) {
    auto c = dev::to_i64(counts);
    const auto cp = dev::to_i64(caps);
    dev::check(adakv_repair_zero_budgets(c.data(), cp.data(), int64_t(c.size())));
    counts = dev::to_size(c);
}

// Layer-wide / per-row selection over ragged f64 rows (one problem).
struct SelectOut {
    std::vector<int32_t> raw, budgets;
    std::vector<std::uint8_t> keep;
};

inline SelectOut select_rows(const WeightRows& rows, std::size_t total, int mode, bool blend, double alpha,
                             bool repair, const std::vector<int32_t>* given, bool streaming = false,
                             std::size_t sink = 0) {
    const std::size_t S = rows.size();
    std::vector<int64_t> off(S + 1, 0);
    for (std::size_t i = 0; i < S; ++i) off[i + 1] = off[i] + int64_t(rows[i].size());
    std::vector<double> flat;
    flat.reserve(std::size_t(off[S]));
    for (const auto& r : rows) {
        for (double x : r)
            if (std::isnan(x)) throw std::invalid_argument("selection: NaN weight");
        flat.insert(flat.end(), r.begin(), r.end());
    }
    const std::size_t N = std::size_t(off[S]);
    dev::Buffer<double> ds(flat.data(), std::max<std::size_t>(N, 1));
    dev::Buffer<int32_t> raw(S), bud(S);
    if (given) bud.upload(given->data(), S);
    dev::Buffer<std::uint8_t> keep(std::max<std::size_t>(N, 1));
    std::size_t ws_bytes = 0;
    dev::check(adakv_segmented_select_workspace(1, int64_t(S), &ws_bytes));
    dev::Buffer<std::uint8_t> ws(ws_bytes);
    adakv_select_config cfg{mode, blend ? 1 : 0, repair ? 1 : 0, streaming ? 1 : 0, alpha, int64_t(sink)};
    dev::check(adakv_segmented_select(ADAKV_F64, 1, int64_t(S), off.data(), ds.get(), int64_t(total), nullptr, &cfg,
                                      raw.get(), bud.get(), keep.get(), nullptr, 0, ws.get(), ws_bytes, nullptr));
    dev::check(adakv_workspace_status(ws.get(), nullptr));
    SelectOut o;
    o.raw = raw.download(S);
    o.budgets = bud.download(S);
    o.keep = keep.download(N);
    return o;
}

}  // namespace detail

/// uniform_allocation (budget.hpp:103-113).
inline BudgetAllocation uniform_allocation(std::size_t total, std::size_t h, std::span<const std::size_t> caps) {
    if (h == 0) throw std::invalid_argument("uniform_allocation: no heads");
    std::vector<int64_t> out(h);
    const auto c = dev::to_i64(caps);
    dev::check(adakv_uniform_allocation(int64_t(total), int64_t(h), c.data(), out.data()));
    return {dev::to_size(out), total};
}
inline BudgetAllocation uniform_allocation(std::size_t total, std::size_t h) {
    return uniform_allocation(total, h, detail::ample_caps(h));
}

/// adaptive_allocation (budget.hpp:118-140): layer-wide radix top-`total` on the device.
inline BudgetAllocation adaptive_allocation(const WeightRows& a, std::size_t total,
                                            TieBreak = TieBreak::by_head_then_position) {
    if (a.empty()) throw std::invalid_argument("adaptive_allocation: no heads");
    std::size_t n = 0;
    for (const auto& r : a) n += r.size();
    if (total > n) throw std::invalid_argument("adaptive_allocation: total exceeds element count");
    const auto o = detail::select_rows(a, total, ADAKV_ALLOC_ADAPTIVE, false, 1.0, false, nullptr);
    return {dev::to_size(o.raw), total};
}

/// safeguard_blend (budget.hpp:145-164).
inline BudgetAllocation safeguard_blend(const BudgetAllocation& adaptive, std::size_t total, std::size_t h,
                                        double alpha, std::span<const std::size_t> caps) {
    if (adaptive.per_head.size() != h) throw std::invalid_argument("safeguard_blend: head count mismatch");
    if (adaptive.total != total) throw std::invalid_argument("safeguard_blend: total mismatch");
    if (!(alpha >= 0.0 && alpha <= 1.0)) throw std::invalid_argument("safeguard_blend: alpha outside [0,1]");
    const auto a = dev::to_i64(adaptive.per_head);
    const auto c = dev::to_i64(caps);
    std::vector<int64_t> out(h);
    dev::check(adakv_safeguard_blend(a.data(), int64_t(adaptive.total), int64_t(total), int64_t(h), alpha, c.data(),
                                     out.data()));
    return {dev::to_size(out), total};
}
inline BudgetAllocation safeguard_blend(const BudgetAllocation& adaptive, std::size_t total, std::size_t h,
                                        double alpha) {
    return safeguard_blend(adaptive, total, h, alpha, detail::ample_caps(h));
}

/// pyramid_layer_budgets (budget.hpp:169-191).
inline std::vector<std::size_t> pyramid_layer_budgets(std::size_t per_layer_avg, std::size_t num_layers,
                                                      double beta_max, double beta_min) {
    std::vector<int64_t> out(std::max<std::size_t>(num_layers, 1));
    dev::check(adakv_pyramid_layer_budgets(int64_t(per_layer_avg), int64_t(num_layers), beta_max, beta_min, out.data()));
    out.resize(num_layers);
    return dev::to_size(out);
}

// --------------------------------------------------------------------------- L3 policies (policies.hpp)
enum class PolicyKind { snapkv, pyramid, ada_snapkv, ada_pyramid, streaming_llm };

inline const char* to_string(PolicyKind k) {
    switch (k) {
        case PolicyKind::snapkv: return "snapkv";
        case PolicyKind::pyramid: return "pyramid";
        case PolicyKind::ada_snapkv: return "ada_snapkv";
        case PolicyKind::ada_pyramid: return "ada_pyramid";
        case PolicyKind::streaming_llm: return "streaming_llm";
    }
    throw std::invalid_argument("to_string: unknown policy kind");
}
inline PolicyKind policy_kind_from_string(const std::string& s) {
    for (auto k : {PolicyKind::snapkv, PolicyKind::pyramid, PolicyKind::ada_snapkv, PolicyKind::ada_pyramid,
                   PolicyKind::streaming_llm})
        if (s == to_string(k)) return k;
    throw std::invalid_argument("unknown policy kind: " + s);
}
inline bool is_adaptive(PolicyKind k) { return k == PolicyKind::ada_snapkv || k == PolicyKind::ada_pyramid; }
inline bool is_pyramid(PolicyKind k) { return k == PolicyKind::pyramid || k == PolicyKind::ada_pyramid; }

struct PolicyConfig {
    PolicyKind kind = PolicyKind::ada_snapkv;
    std::size_t window_size = 32;
    std::size_t pool_kernel = 7;
    double alpha = 0.2;
    std::size_t sink_tokens = 4;
    std::size_t gqa_group_size = 1;
    bool scale = true;
    void validate() const {
        if (window_size < 1) throw std::invalid_argument("PolicyConfig: window_size < 1");
        if (pool_kernel % 2 == 0 || pool_kernel == 0) throw std::invalid_argument("PolicyConfig: pool_kernel must be odd");
        if (!(alpha >= 0.0 && alpha <= 1.0)) throw std::invalid_argument("PolicyConfig: alpha outside [0,1]");
        if (gqa_group_size == 0) throw std::invalid_argument("PolicyConfig: zero group size");
    }
};

using ObservationScores = std::vector<std::vector<double>>;

/// topk_decision (policies.hpp:80-93): keep the k largest, ties to the lowest position.
inline std::vector<std::uint8_t> topk_decision(std::span<const double> a, std::size_t k,
                                               TieBreak = TieBreak::by_head_then_position) {
    if (k > a.size()) throw std::invalid_argument("topk_decision: k exceeds length");
    if (a.empty()) return {};
    const std::vector<int32_t> given{int32_t(k)};
    const auto o = detail::select_rows(WeightRows{WeightRow(a.begin(), a.end())}, 0, ADAKV_ALLOC_GIVEN, false, 1.0,
                                       false, &given);
    return o.keep;
}

/// streaming_llm_decision (policies.hpp:159-165): positions [0, sink) and [n - recent, n).
inline std::vector<std::uint8_t> streaming_llm_decision(std::size_t n, std::size_t sink, std::size_t recent) {
    if (n == 0) return {};
    const std::size_t s = std::min(sink, n), r = std::min(recent, n);
    const bool overlap = s + r >= n;
    const std::vector<int32_t> given{int32_t(overlap ? n : s + r)};
    const auto o = detail::select_rows(WeightRows{WeightRow(n, 0.0)}, 0, ADAKV_ALLOC_GIVEN, false, 1.0, false, &given,
                                       !overlap, s);
    return o.keep;
}

/// window_scores (policies.hpp:119-132) on the device (fp64 path).
inline std::vector<double> window_scores(const Matrix& window_queries, const Matrix& outside_keys,
                                         std::size_t pool_kernel, bool scale = true) {
    if (window_queries.rows() == 0) throw std::invalid_argument("window_scores: empty window");
    if (outside_keys.rows() == 0) throw std::invalid_argument("attention_weights: empty key set");
    if (window_queries.cols() != outside_keys.cols()) throw std::invalid_argument("attention_weights: head dim mismatch");
    if (pool_kernel % 2 == 0 || pool_kernel == 0) throw std::invalid_argument("maxpool: kernel must be odd");
    const std::size_t m = window_queries.rows(), n = outside_keys.rows(), d = outside_keys.cols();
    // device layout [1 group][n + m rows][d]: outside rows then m (unused) window rows
    std::vector<double> kbuf((n + m) * d, 0.0);
    std::copy(outside_keys.values().begin(), outside_keys.values().end(), kbuf.begin());
    dev::Buffer<double> dq(window_queries.values().data(), m * d), dk(kbuf.data(), kbuf.size()), ds(n);
    adakv_layer_shape shape{1, 1, 1, int64_t(m), int64_t(n), int64_t(d)};
    std::size_t wsb = 0;
    dev::check(adakv_window_scores_workspace(ADAKV_F64, &shape, &wsb));
    dev::Buffer<std::uint8_t> ws(wsb);
    dev::check(adakv_window_scores(ADAKV_F64, &shape, int64_t(pool_kernel), scale ? 1 : 0, dq.get(), dk.get(), nullptr,
                                   ds.get(), ws.get(), wsb, nullptr));
    return ds.download(n);
}

/// group_mean_scores (policies.hpp:136-156) on the device.
inline ObservationScores group_mean_scores(const ObservationScores& scores, std::size_t group_size) {
    if (group_size == 0) throw std::invalid_argument("group_mean_scores: zero group size");
    if (scores.size() % group_size != 0)
        throw std::invalid_argument("group_mean_scores: head count not divisible by group size");
    const std::size_t groups = scores.size() / group_size;
    ObservationScores out(groups);
    for (std::size_t gi = 0; gi < groups; ++gi) {
        const std::size_t n = scores[gi * group_size].size();
        std::vector<double> flat;
        for (std::size_t k = 0; k < group_size; ++k) {
            const auto& s = scores[gi * group_size + k];
            if (s.size() != n) throw std::invalid_argument("group_mean_scores: member length mismatch");
            flat.insert(flat.end(), s.begin(), s.end());
        }
        if (n == 0) continue;
        dev::Buffer<double> ds(flat.data(), flat.size()), dout(n);
        dev::check(adakv_group_mean_scores_f64(ds.get(), int64_t(group_size), int64_t(n), int64_t(group_size),
                                               dout.get(), nullptr));
        out[gi] = dout.download(n);
    }
    return out;
}

struct EvictLayerResult {
    LayerCache retained;
    EvictionDecision decision;    // over outside positions, one entry per head
    BudgetAllocation allocation;  // outside budget split, one entry per KV group
    ObservationScores scores;     // pooled observation scores, one entry per KV group
};

/// evict_layer (policies.hpp:204-293): the whole compression pass on the device.
inline EvictLayerResult evict_layer(const LayerCache& cache_outside, const LayerCache& window_cache,
                                    const Matrix& window_embeddings, const LayerParams& params,
                                    std::size_t layer_budget, const PolicyConfig& config) {
    config.validate();
    params.validate();
    cache_outside.validate();
    window_cache.validate();
    const std::size_t h = params.head_count();
    if (cache_outside.head_count() != h || window_cache.head_count() != h)
        throw std::invalid_argument("evict_layer: head count mismatch");
    const std::size_t g = config.gqa_group_size;
    if (h % g != 0) throw std::invalid_argument("evict_layer: head count not divisible by group");
    const std::size_t groups = h / g;
    const std::size_t m = window_embeddings.rows();
    if (m == 0) throw std::invalid_argument("evict_layer: empty window");
    if (window_embeddings.cols() != params.embed_dim()) throw std::invalid_argument("evict_layer: embedding width mismatch");
    for (std::size_t i = 0; i < h; ++i) {
        if (window_cache.heads[i].length() != m) throw std::invalid_argument("evict_layer: window cache length mismatch");
        if (cache_outside.heads[i].length() != cache_outside.heads[(i / g) * g].length())
            throw std::invalid_argument("evict_layer: unequal lengths within a group");
    }
    if (layer_budget < m * groups + groups) throw std::invalid_argument("evict_layer: budget below the window-plus-one floor");
    const std::size_t n_o = cache_outside.heads[0].length();
    for (std::size_t gi = 0; gi < groups; ++gi) {
        if (cache_outside.heads[gi * g].length() == 0) throw std::invalid_argument("evict_layer: empty outside cache head");
        if (cache_outside.heads[gi * g].length() != n_o)
            throw std::invalid_argument("evict_layer (B200): all KV groups must share one outside length");
        for (std::size_t k = 1; k < g; ++k) {
            const auto& a = cache_outside.heads[gi * g], & b = cache_outside.heads[gi * g + k];
            const auto& wa = window_cache.heads[gi * g], & wb = window_cache.heads[gi * g + k];
            if (!(a.keys == b.keys && a.values == b.values && wa.keys == wb.keys && wa.values == wb.values))
                throw std::invalid_argument("evict_layer (B200): the heads of a KV group must share K/V");
        }
    }
    const std::size_t outside_budget = layer_budget - m * groups;
    if (outside_budget > groups * n_o) throw std::invalid_argument("apportion: total exceeds capacity");
    const std::size_t d = params.head_dim(), D = params.embed_dim();
    // queries: Q_i = X W_q,i on the device (policies.hpp:243)
    std::vector<double> wq;
    wq.reserve(h * D * d);
    for (const auto& hp : params.heads) wq.insert(wq.end(), hp.wq.values().begin(), hp.wq.values().end());
    dev::Buffer<double> dx(window_embeddings.values().data(), m * D), dwq(wq.data(), wq.size()), dq(h * m * d);
    dev::check(adakv_project_queries_f64(dx.get(), dwq.get(), int64_t(h), int64_t(m), int64_t(D), int64_t(d), dq.get(),
                                         nullptr));
    // prompt K/V per group: outside rows then window rows
    const std::size_t n = n_o + m;
    std::vector<double> kh(groups * n * d), vh(groups * n * d);
    for (std::size_t gi = 0; gi < groups; ++gi) {
        const auto& o = cache_outside.heads[gi * g];
        const auto& w = window_cache.heads[gi * g];
        std::copy(o.keys.values().begin(), o.keys.values().end(), kh.begin() + gi * n * d);
        std::copy(w.keys.values().begin(), w.keys.values().end(), kh.begin() + (gi * n + n_o) * d);
        std::copy(o.values.values().begin(), o.values.values().end(), vh.begin() + gi * n * d);
        std::copy(w.values.values().begin(), w.values.values().end(), vh.begin() + (gi * n + n_o) * d);
    }
    dev::Buffer<double> dk(kh.data(), kh.size()), dv(vh.data(), vh.size());
    adakv_layer_shape shape{1, int64_t(h), int64_t(groups), int64_t(m), int64_t(n_o), int64_t(d)};
    adakv_policy_config cfg{int32_t(config.kind), config.scale ? 1 : 0, int64_t(config.window_size),
                            int64_t(config.pool_kernel), config.alpha, int64_t(config.sink_tokens), int64_t(g)};
    const int64_t rows = adakv_cache_rows(&shape, int64_t(layer_budget), nullptr, 0);
    dev::Buffer<double> kc(std::size_t(rows) * d), vc(std::size_t(rows) * d), gsc(groups * n_o);
    dev::Buffer<int32_t> ss(groups), sl(groups), bud(groups);
    dev::Buffer<std::uint8_t> keep(groups * n_o);
    std::size_t wsb = 0;
    dev::check(adakv_compress_workspace(ADAKV_F64, &shape, &cfg, &wsb));
    dev::Buffer<std::uint8_t> ws(wsb);
    dev::check(adakv_compress(ADAKV_F64, &shape, &cfg, int64_t(layer_budget), nullptr, dq.get(), dk.get(), dv.get(), 0,
                              kc.get(), vc.get(), ss.get(), sl.get(), nullptr, bud.get(), gsc.get(), keep.get(), ws.get(), wsb,
                              nullptr));
    dev::check(adakv_workspace_status(ws.get(), nullptr));
    const auto h_bud = bud.download(groups);
    const auto h_keep = keep.download(groups * n_o);
    const auto h_sc = gsc.download(groups * n_o);
    const auto h_ss = ss.download(groups), h_sl = sl.download(groups);
    const auto h_k = kc.download(std::size_t(rows) * d), h_v = vc.download(std::size_t(rows) * d);
    EvictLayerResult res;
    res.allocation = {dev::to_size(h_bud), outside_budget};
    res.scores.resize(groups);
    res.decision.retain.resize(h);
    res.retained.heads.resize(h);
    for (std::size_t gi = 0; gi < groups; ++gi) {
        res.scores[gi].assign(h_sc.begin() + gi * n_o, h_sc.begin() + (gi + 1) * n_o);
        const std::vector<std::uint8_t> kp(h_keep.begin() + gi * n_o, h_keep.begin() + (gi + 1) * n_o);
        Matrix keys(std::size_t(h_sl[gi]), d), vals(std::size_t(h_sl[gi]), d);
        std::copy(h_k.begin() + std::size_t(h_ss[gi]) * d, h_k.begin() + std::size_t(h_ss[gi] + h_sl[gi]) * d,
                  keys.values().begin());
        std::copy(h_v.begin() + std::size_t(h_ss[gi]) * d, h_v.begin() + std::size_t(h_ss[gi] + h_sl[gi]) * d,
                  vals.values().begin());
        for (std::size_t k = 0; k < g; ++k) {
            res.decision.retain[gi * g + k] = kp;
            res.retained.heads[gi * g + k] = {keys, vals};
        }
    }
    return res;
}

/// evict_rows (policies.hpp:298-323): weights-only theory mode (alpha defaults to 1.0).
inline std::pair<EvictionDecision, BudgetAllocation> evict_rows(const WeightRows& weights, std::size_t total_budget,
                                                                bool adaptive, double alpha = 1.0) {
    const std::size_t h = weights.size();
    if (h == 0) throw std::invalid_argument("evict_rows: no heads");
    std::size_t n = 0;
    for (const auto& r : weights) {
        if (r.empty()) throw std::invalid_argument("evict_rows: empty head");
        n += r.size();
    }
    if (total_budget < h) throw std::invalid_argument("evict_rows: budget below one per head");
    if (total_budget > n) throw std::invalid_argument(adaptive ? "adaptive_allocation: total exceeds element count"
                                                               : "apportion: total exceeds capacity");
    if (adaptive && !(alpha >= 0.0 && alpha <= 1.0)) throw std::invalid_argument("safeguard_blend: alpha outside [0,1]");
    const auto o = detail::select_rows(weights, total_budget, adaptive ? ADAKV_ALLOC_ADAPTIVE : ADAKV_ALLOC_UNIFORM,
                                       adaptive, alpha, true, nullptr);
    EvictionDecision dec;
    dec.retain.resize(h);
    std::size_t off = 0;
    for (std::size_t i = 0; i < h; ++i) {
        dec.retain[i].assign(o.keep.begin() + off, o.keep.begin() + off + weights[i].size());
        off += weights[i].size();
    }
    return {std::move(dec), BudgetAllocation{dev::to_size(o.budgets), total_budget}};
}

// --------------------------------------------------------------------------- L3 layout (flat_cache.hpp)
struct FlattenedCache {
    std::vector<double> data;  // per head: K rows then V rows
    std::vector<std::size_t> offsets, lengths;
    std::size_t d_h = 0;
    std::size_t head_count() const { return lengths.size(); }
    std::size_t total_elements() const {
        std::size_t n = 0;
        for (auto l : lengths) n += l;
        return n;
    }
};

struct CacheStats {
    std::size_t total_elements = 0;
    std::size_t bytes = 0;
    std::vector<std::size_t> per_head;
};

/// flatten (flat_cache.hpp:44-66): layout conversion, offsets count rows.
inline FlattenedCache flatten(const LayerCache& cache) {
    cache.validate();
    FlattenedCache fc;
    std::size_t off = 0;
    for (const auto& head : cache.heads) {
        if (head.keys.cols() != cache.heads.front().keys.cols()) throw std::invalid_argument("flatten: inconsistent head widths");
        fc.offsets.push_back(off);
        fc.lengths.push_back(head.length());
        off += head.length();
    }
    fc.d_h = cache.heads.empty() ? 0 : cache.heads.front().keys.cols();
    fc.data.reserve(2 * off * fc.d_h);
    for (const auto& head : cache.heads) {
        fc.data.insert(fc.data.end(), head.keys.values().begin(), head.keys.values().end());
        fc.data.insert(fc.data.end(), head.values.values().begin(), head.values.values().end());
    }
    return fc;
}

/// head_slice (flat_cache.hpp:69-81).
inline HeadKV head_slice(const FlattenedCache& fc, std::size_t i) {
    if (i >= fc.head_count()) throw std::out_of_range("head_slice: head index out of range");
    const std::size_t n = fc.lengths[i], base = fc.offsets[i] * 2 * fc.d_h;
    Matrix keys(n, fc.d_h), values(n, fc.d_h);
    std::copy(fc.data.begin() + base, fc.data.begin() + base + n * fc.d_h, keys.values().begin());
    std::copy(fc.data.begin() + base + n * fc.d_h, fc.data.begin() + base + 2 * n * fc.d_h, values.values().begin());
    return {std::move(keys), std::move(values)};
}

inline LayerCache unflatten(const FlattenedCache& fc) {
    LayerCache c;
    for (std::size_t i = 0; i < fc.head_count(); ++i) c.heads.push_back(head_slice(fc, i));
    return c;
}

/// select_and_compact (flat_cache.hpp:92-120): the compaction runs on the device.
inline FlattenedCache select_and_compact(const FlattenedCache& fc, const EvictionDecision& decision) {
    if (decision.head_count() != fc.head_count()) throw std::invalid_argument("select_and_compact: head count mismatch");
    const std::size_t h = fc.head_count(), d = fc.d_h;
    FlattenedCache out;
    out.d_h = d;
    std::vector<int64_t> off(h + 1, 0), out_off(h + 1, 0);
    std::vector<std::uint8_t> mask;
    std::vector<double> k, v;
    for (std::size_t i = 0; i < h; ++i) {
        if (decision.retain[i].size() != fc.lengths[i]) throw std::invalid_argument("select_and_compact: decision length mismatch");
        const std::size_t kept = decision.retained_count(i);
        out.offsets.push_back(std::size_t(out_off[i]));
        out.lengths.push_back(kept);
        out_off[i + 1] = out_off[i] + int64_t(kept);
        off[i + 1] = off[i] + int64_t(fc.lengths[i]);
        mask.insert(mask.end(), decision.retain[i].begin(), decision.retain[i].end());
        const std::size_t base = fc.offsets[i] * 2 * d, n = fc.lengths[i];
        k.insert(k.end(), fc.data.begin() + base, fc.data.begin() + base + n * d);
        v.insert(v.end(), fc.data.begin() + base + n * d, fc.data.begin() + base + 2 * n * d);
    }
    const std::size_t total = std::size_t(out_off[h]);
    out.data.resize(2 * total * d);
    if (total == 0 || d == 0) return out;
    dev::Buffer<std::uint8_t> dm(mask.data(), mask.size());
    dev::Buffer<int64_t> doff(off.data(), off.size()), doo(out_off.data(), out_off.size());
    dev::Buffer<double> dk(k.data(), k.size()), dv(v.data(), v.size()), ok(total * d), ov(total * d);
    dev::check(adakv_compact_rows_f64(int64_t(h), dm.get(), doff.get(), dk.get(), dv.get(), int64_t(d), doo.get(),
                                      ok.get(), ov.get(), nullptr));
    const auto hk = ok.download(total * d), hv = ov.download(total * d);
    for (std::size_t i = 0; i < h; ++i) {
        const std::size_t n = out.lengths[i], src = std::size_t(out_off[i]) * d, dst = out.offsets[i] * 2 * d;
        std::copy(hk.begin() + src, hk.begin() + src + n * d, out.data.begin() + dst);
        std::copy(hv.begin() + src, hv.begin() + src + n * d, out.data.begin() + dst + n * d);
    }
    return out;
}

/// memory_footprint (flat_cache.hpp:122-129).
inline CacheStats memory_footprint(const FlattenedCache& fc, std::size_t bytes_per_value = sizeof(double)) {
    CacheStats s;
    s.per_head = fc.lengths;
    s.total_elements = fc.total_elements();
    s.bytes = s.total_elements * fc.d_h * 2 * bytes_per_value;
    return s;
}

// AKVC v1 persistence (flat_cache.hpp:131-178): "AKVC", u32 version, u32 h, u32 d_h,
// u64 lengths[h], then the data as little-endian f64.
inline constexpr std::uint32_t kAkvcVersion = 1;

namespace detail {
inline void put_le(std::ostream& os, std::uint64_t v, int nbytes) {
    unsigned char b[8];
    for (int i = 0; i < nbytes; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
    os.write(reinterpret_cast<const char*>(b), nbytes);
}
inline std::uint64_t get_le(std::istream& is, int nbytes) {
    unsigned char b[8];
    if (!is.read(reinterpret_cast<char*>(b), nbytes)) throw FormatError("unexpected end of file");
    std::uint64_t v = 0;
    for (int i = 0; i < nbytes; ++i) v |= std::uint64_t(b[i]) << (8 * i);
    return v;
}
}  // namespace detail

inline void save_flattened(const FlattenedCache& fc, std::ostream& os) {
    os.write("AKVC", 4);
    detail::put_le(os, kAkvcVersion, 4);
    detail::put_le(os, fc.head_count(), 4);
    detail::put_le(os, fc.d_h, 4);
    for (auto l : fc.lengths) detail::put_le(os, l, 8);
    for (double x : fc.data) {
        std::uint64_t u;
        std::memcpy(&u, &x, 8);
        detail::put_le(os, u, 8);
    }
    if (!os) throw IoError("save_flattened: write failed");
}

inline FlattenedCache load_flattened(std::istream& is) {
    char magic[4];
    if (!is.read(magic, 4)) throw FormatError("load_flattened: truncated header");
    if (std::string(magic, 4) != "AKVC") throw FormatError("load_flattened: bad magic");
    const auto version = detail::get_le(is, 4);
    if (version != kAkvcVersion) throw FormatError("load_flattened: unsupported version " + std::to_string(version));
    const auto h = detail::get_le(is, 4), d_h = detail::get_le(is, 4);
    FlattenedCache fc;
    fc.d_h = std::size_t(d_h);
    std::size_t off = 0;
    for (std::uint64_t i = 0; i < h; ++i) {
        fc.offsets.push_back(off);
        const auto l = std::size_t(detail::get_le(is, 8));
        fc.lengths.push_back(l);
        off += l;
    }
    fc.data.resize(2 * off * fc.d_h);
    for (double& x : fc.data) {
        const std::uint64_t u = detail::get_le(is, 8);
        std::memcpy(&x, &u, 8);
    }
    return fc;
}

inline void save_flattened_file(const FlattenedCache& fc, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open for writing: " + path);
    save_flattened(fc, os);
}

inline FlattenedCache load_flattened_file(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoError("cannot open for reading: " + path);
    return load_flattened(is);
}

}  // namespace adakv_b200
