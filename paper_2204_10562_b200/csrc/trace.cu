// Host-side schedule trace writer (reference fileio.py:170-188, format_number
// fileio.py:32-38): "# makespan X", the column header, one CSV row per event
// and one "allreduce,0,allreduce_stage<n>,start,end" row per window.  Every
// number is "%.9g" (glibc and CPython both round correctly, so the bytes are
// the reference's); the first non-finite value in output order is an error.
//
// Rows are formatted by up to `nthreads` host threads into private buffers
// and concatenated in order, so the text is identical for any thread count.
// Included from capi.cu (needs fail()).

#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// Python's str() of a non-finite float, for the error text.
const char* nonfinite_text(double x) { return std::isnan(x) ? "nan" : (x > 0 ? "inf" : "-inf"); }

struct RowWriter {
    char* p;
    void put(const char* s) {
        size_t n = strlen(s);
        memcpy(p, s, n);
        p += n;
    }
    void ch(char c) { *p++ = c; }
    void num(double x) { p += snprintf(p, 32, "%.9g", x); }
    void integer(long long v) { p += snprintf(p, 24, "%lld", v); }
};

}  // namespace

extern "C" int pp_format_trace(int64_t n_events, const int32_t* ev_m, const int32_t* ev_pos,
                               const double* ev_start, const double* ev_end, const char* const* res_names,
                               const char* const* labels, int32_t n_names, int32_t n_ar,
                               const int32_t* ar_stage, const double* ar_start, const double* ar_end,
                               double makespan, char* out, int64_t cap, int64_t* out_len, int32_t nthreads) {
    if (n_events < 0 || n_ar < 0 || n_names < 0 || !out || !out_len)
        return fail(PP_EINVAL, "pp_format_trace: bad arguments");
    // non-finite check in output order: makespan, events, windows
    if (!std::isfinite(makespan))
        return fail(PP_EINVAL, "non-finite number in output: %s", nonfinite_text(makespan));
    size_t name_max = 0;
    for (int32_t q = 0; q < n_names; ++q) {
        if (res_names[q]) name_max = std::max(name_max, strlen(res_names[q]));
        if (labels[q]) name_max = std::max(name_max, strlen(labels[q]));
    }
    for (int64_t k = 0; k < n_events; ++k) {
        int32_t q = ev_pos[k];
        if (q < 0 || q >= n_names || !res_names[q] || !labels[q])
            return fail(PP_EINVAL, "pp_format_trace: event %lld has no name (index %d)", (long long)k, q);
        if (!std::isfinite(ev_start[k]))
            return fail(PP_EINVAL, "non-finite number in output: %s", nonfinite_text(ev_start[k]));
        if (!std::isfinite(ev_end[k]))
            return fail(PP_EINVAL, "non-finite number in output: %s", nonfinite_text(ev_end[k]));
    }
    for (int32_t w = 0; w < n_ar; ++w) {
        if (!std::isfinite(ar_start[w]))
            return fail(PP_EINVAL, "non-finite number in output: %s", nonfinite_text(ar_start[w]));
        if (!std::isfinite(ar_end[w]))
            return fail(PP_EINVAL, "non-finite number in output: %s", nonfinite_text(ar_end[w]));
    }
    // per-row upper bound: 2 names, an int (<= 11), two numbers (<= 24), 4 commas, '\n'
    const size_t row_max = 2 * name_max + 11 + 2 * 24 + 5 + 32;
    static const char kHeader[] = "resource,microbatch,block,start,end\n";
    const size_t head_max = 11 + 24 + 1 + sizeof(kHeader);

    int T = std::max(1, std::min<int>(nthreads, 64));
    if (n_events < 4096) T = 1;
    std::vector<std::vector<char>> bufs(T);
    std::vector<size_t> lens(T, 0);
    auto work = [&](int t) {
        int64_t lo = n_events * t / T, hi = n_events * (t + 1) / T;
        bufs[t].resize((size_t)(hi - lo) * row_max + 1);
        RowWriter w{bufs[t].data()};
        for (int64_t k = lo; k < hi; ++k) {
            int32_t q = ev_pos[k];
            w.put(res_names[q]);
            w.ch(',');
            w.integer(ev_m[k]);
            w.ch(',');
            w.put(labels[q]);
            w.ch(',');
            w.num(ev_start[k]);
            w.ch(',');
            w.num(ev_end[k]);
            w.ch('\n');
        }
        lens[t] = (size_t)(w.p - bufs[t].data());
    };
    if (T == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
    }
    std::vector<char> tail((size_t)n_ar * (40 + 2 * 24 + 16) + 1);
    RowWriter tw{tail.data()};
    for (int32_t w = 0; w < n_ar; ++w) {
        tw.put("allreduce,0,allreduce_stage");
        tw.integer(ar_stage[w]);
        tw.ch(',');
        tw.num(ar_start[w]);
        tw.ch(',');
        tw.num(ar_end[w]);
        tw.ch('\n');
    }
    std::vector<char> head(head_max);
    RowWriter hw{head.data()};
    hw.put("# makespan ");
    hw.num(makespan);
    hw.ch('\n');
    hw.put(kHeader);

    size_t total = (size_t)(hw.p - head.data()) + (size_t)(tw.p - tail.data());
    for (int t = 0; t < T; ++t) total += lens[t];
    *out_len = (int64_t)total;
    if ((int64_t)total > cap) return fail(PP_EINVAL, "pp_format_trace: output needs %zu bytes, cap %lld", total,
                                          (long long)cap);
    char* o = out;
    memcpy(o, head.data(), (size_t)(hw.p - head.data()));
    o += hw.p - head.data();
    for (int t = 0; t < T; ++t) {
        memcpy(o, bufs[t].data(), lens[t]);
        o += lens[t];
    }
    memcpy(o, tail.data(), (size_t)(tw.p - tail.data()));
    return 0;
}
