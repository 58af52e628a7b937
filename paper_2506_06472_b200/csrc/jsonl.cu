// jsonl.cu — multi-threaded host parser of the reference trace JSONL format
// (trace.py:160-275 parse_trace; writer trace.py:278-301) straight into the
// column form libtio and the device path consume.
//
// Fast path only: any line that is not a well-formed record of the format
// (unknown / missing keys, non-integer or non-int64 numbers, bad kinds, kernel
// after tensor records, ...) makes tio_trace_parse return TIO_ERR_INVALID with
// the 1-based line number; the Python layer then re-parses with the
// reference-exact parser to raise the reference's TraceParseError text.
// Model invariants (validate_trace, trace.py:125-157) are checked by the
// caller on the columns.
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace tio {
namespace {

constexpr int64_t NONE_I64 = INT64_MIN;

struct Cursor {
    const char *p, *e;
    bool ok = true;
    void ws() { while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p; }
    bool lit(char c) { ws(); if (p < e && *p == c) { ++p; return true; } return false; }
    bool word(const char *w) {
        ws();
        size_t n = strlen(w);
        if ((size_t)(e - p) >= n && memcmp(p, w, n) == 0) { p += n; return true; }
        return false;
    }
    // JSON string: returns the raw contents (escapes kept); false on error
    bool str(const char **s, size_t *n, bool *escaped) {
        ws();
        if (p >= e || *p != '"') return false;
        ++p;
        const char *b = p;
        *escaped = false;
        while (p < e && *p != '"') {
            if (*p == '\\') { *escaped = true; ++p; if (p >= e) return false; }
            else if ((unsigned char)*p < 0x20) return false;
            ++p;
        }
        if (p >= e) return false;
        *s = b; *n = (size_t)(p - b);
        ++p;
        return true;
    }
    // JSON integer in int64 (no fraction / exponent); false otherwise
    bool i64(int64_t *v) {
        ws();
        bool neg = false;
        if (p < e && *p == '-') { neg = true; ++p; }
        if (p >= e || *p < '0' || *p > '9') return false;
        if (*p == '0' && p + 1 < e && p[1] >= '0' && p[1] <= '9') return false;
        unsigned long long acc = 0;
        while (p < e && *p >= '0' && *p <= '9') {
            unsigned d = (unsigned)(*p - '0');
            if (acc > (ULLONG_MAX - d) / 10) return false;
            acc = acc * 10 + d;
            ++p;
        }
        if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) return false;
        if (neg ? acc > 9223372036854775808ull : acc > 9223372036854775807ull) return false;
        *v = neg ? (int64_t)(0 - acc) : (int64_t)acc;
        return true;
    }
    bool i64_or_null(int64_t *v) {
        if (word("null")) { *v = NONE_I64; return true; }
        return i64(v);
    }
};

struct Part {
    // kernels
    std::vector<int64_t> k_index, k_dur, k_stage, k_layer;
    std::vector<std::string> k_name;       // raw JSON string contents
    std::vector<uint8_t> k_name_esc;
    // tensors
    std::vector<int64_t> t_id, t_size, t_layer, t_count, acc;
    std::vector<int8_t> t_kind;
    int64_t first_tensor_line = -1, last_kernel_line = -1;
    int64_t err_line = -1;
};

// one record line; returns false on any deviation from the fast format
bool parse_record(Cursor &c, Part &o, int64_t lineno) {
    if (!c.lit('{')) return false;
    const char *k; size_t kn; bool esc;
    if (!c.str(&k, &kn, &esc) || esc || !c.lit(':') || !c.lit('{')) return false;
    const bool is_kernel = kn == 6 && memcmp(k, "kernel", 6) == 0;
    const bool is_tensor = kn == 6 && memcmp(k, "tensor", 6) == 0;
    if (!is_kernel && !is_tensor) return false;
    unsigned seen = 0;
    int64_t a = 0, b = 0, st = NONE_I64, ly = NONE_I64;
    int8_t kind = -1;
    const char *nm = nullptr; size_t nml = 0; bool nesc = false;
    size_t acc0 = o.acc.size();
    if (!c.lit('}')) {
        do {
            const char *f; size_t fn; bool fe;
            if (!c.str(&f, &fn, &fe) || fe || !c.lit(':')) return false;
            auto is = [&](const char *w) { return fn == strlen(w) && memcmp(f, w, fn) == 0; };
            unsigned bit;
            if (is_kernel) {
                if (is("index")) { bit = 1; if (!c.i64(&a)) return false; }
                else if (is("name")) { bit = 2; if (!c.str(&nm, &nml, &nesc)) return false; }
                else if (is("duration_us")) { bit = 4; if (!c.i64(&b)) return false; }
                else if (is("stage")) { bit = 8; if (!c.i64_or_null(&st)) return false; }
                else if (is("layer")) { bit = 16; if (!c.i64_or_null(&ly)) return false; }
                else return false;
            } else {
                if (is("id")) { bit = 1; if (!c.i64(&a)) return false; }
                else if (is("size_bytes")) { bit = 2; if (!c.i64(&b)) return false; }
                else if (is("kind")) {
                    bit = 4;
                    const char *s; size_t sn; bool se;
                    if (!c.str(&s, &sn, &se) || se) return false;
                    if (sn == 12 && memcmp(s, "intermediate", 12) == 0) kind = 0;
                    else if (sn == 6 && memcmp(s, "global", 6) == 0) kind = 1;
                    else return false;
                } else if (is("accesses")) {
                    bit = 8;
                    if (!c.lit('[')) return false;
                    if (!c.lit(']')) {
                        do {
                            int64_t v;
                            if (!c.i64(&v)) return false;
                            o.acc.push_back(v);
                        } while (c.lit(','));
                        if (!c.lit(']')) return false;
                    }
                } else if (is("layer")) { bit = 16; if (!c.i64_or_null(&ly)) return false; }
                else return false;
            }
            if (seen & bit) return false;            // duplicate key: let the reference parser decide
            seen |= bit;
        } while (c.lit(','));
        if (!c.lit('}')) return false;
    }
    if (!c.lit('}')) return false;
    c.ws();
    if (c.p != c.e) return false;
    if (is_kernel) {
        if ((seen & 7) != 7) return false;
        if (o.first_tensor_line >= 0) return false;   // kernel after tensor records
        o.k_index.push_back(a); o.k_dur.push_back(b); o.k_stage.push_back(st); o.k_layer.push_back(ly);
        o.k_name.emplace_back(nm, nml);
        o.k_name_esc.push_back(nesc ? 1 : 0);
        o.last_kernel_line = lineno;
    } else {
        if ((seen & 15) != 15) { o.acc.resize(acc0); return false; }
        o.t_id.push_back(a); o.t_size.push_back(b); o.t_kind.push_back(kind); o.t_layer.push_back(ly);
        o.t_count.push_back((int64_t)(o.acc.size() - acc0));
        if (o.first_tensor_line < 0) o.first_tensor_line = lineno;
    }
    return true;
}

void parse_range(const char *b, const char *e, int64_t first_line, Part *o) {
    int64_t lineno = first_line;
    const char *p = b;
    while (p < e) {
        const char *nl = (const char *)memchr(p, '\n', (size_t)(e - p));
        const char *le = nl ? nl : e;
        Cursor c{p, le};
        c.ws();
        if (c.p != c.e && !parse_record(c, *o, lineno)) { o->err_line = lineno; return; }
        p = nl ? nl + 1 : e;
        ++lineno;
    }
}

}  // namespace
}  // namespace tio

using namespace tio;

struct tio_parsed_trace {
    std::vector<int64_t> k_index, k_dur, k_stage, k_layer, t_id, t_size, t_layer, ptr, acc;
    std::vector<int32_t> k_code;
    std::vector<int8_t> t_kind;
    std::string names;          // name table: raw JSON string contents joined with '\n'-free separators
    std::vector<int64_t> name_off;
    std::vector<uint8_t> name_esc;
    std::string meta;           // raw JSON text of the header's meta object
};

// header: {"version": 1, "meta": {...}} (keys in any order, meta optional)
static bool parse_header(const char *b, const char *e, std::string *meta) {
    Cursor c{b, e};
    if (!c.lit('{')) return false;
    bool ver = false;
    *meta = "{}";
    if (!c.lit('}')) {
        do {
            const char *f; size_t fn; bool fe;
            if (!c.str(&f, &fn, &fe) || fe || !c.lit(':')) return false;
            if (fn == 7 && memcmp(f, "version", 7) == 0) {
                int64_t v;
                if (!c.i64(&v) || v != 1) return false;
                ver = true;
            } else if (fn == 4 && memcmp(f, "meta", 4) == 0) {
                // raw object text: balanced braces outside strings
                c.ws();
                if (c.p >= c.e || *c.p != '{') return false;
                const char *s = c.p;
                int depth = 0;
                bool in_str = false;
                for (; c.p < c.e; ++c.p) {
                    char ch = *c.p;
                    if (in_str) { if (ch == '\\') ++c.p; else if (ch == '"') in_str = false; continue; }
                    if (ch == '"') in_str = true;
                    else if (ch == '{' || ch == '[') ++depth;
                    else if (ch == '}' || ch == ']') { if (--depth == 0) { ++c.p; break; } }
                }
                if (depth != 0) return false;
                meta->assign(s, (size_t)(c.p - s));
            } else {
                return false;
            }
        } while (c.lit(','));
        if (!c.lit('}')) return false;
    }
    c.ws();
    return ver && c.p == c.e;
}

extern "C" int tio_trace_parse(const char *buf, size_t len, int threads, tio_parsed_trace **out,
                               int64_t *err_line) {
    if (!buf || !out) return fail(TIO_ERR_INVALID, "null argument");
    *out = nullptr;
    if (err_line) *err_line = 0;
    const char *e = buf + len;
    const char *nl = (const char *)memchr(buf, '\n', len);
    const char *h_end = nl ? nl : e;
    std::string meta;
    if (!parse_header(buf, h_end, &meta)) {
        if (err_line) *err_line = 1;
        return fail(TIO_ERR_INVALID, "header line not in the fast format");
    }
    const char *body = nl ? nl + 1 : e;
    // split the body into chunks at line boundaries
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    if (threads > 64) threads = 64;
    const size_t blen = (size_t)(e - body);
    if (blen < (1u << 20)) threads = 1;
    std::vector<const char *> cut{body};
    for (int i = 1; i < threads; ++i) {
        const char *q = body + blen * i / threads;
        if (q < cut.back()) q = cut.back();
        const char *n2 = (const char *)memchr(q, '\n', (size_t)(e - q));
        cut.push_back(n2 ? n2 + 1 : e);
    }
    cut.push_back(e);
    std::vector<int64_t> first_line(cut.size() - 1, 2);
    for (size_t i = 1; i + 1 < cut.size(); ++i) {
        int64_t n = 0;
        for (const char *q = cut[i - 1]; q < cut[i]; ++q) n += *q == '\n';
        first_line[i] = first_line[i - 1] + n;
    }
    std::vector<Part> parts(cut.size() - 1);
    std::vector<std::thread> pool;
    for (size_t i = 0; i < parts.size(); ++i)
        pool.emplace_back(parse_range, cut[i], cut[i + 1], first_line[i], &parts[i]);
    for (auto &t : pool) t.join();
    int64_t bad = 0;
    bool saw_tensor = false;
    for (auto &pt : parts) {
        if (pt.err_line >= 0) { bad = pt.err_line; break; }
        if (saw_tensor && pt.last_kernel_line >= 0) { bad = pt.last_kernel_line; break; }
        if (pt.first_tensor_line >= 0) saw_tensor = true;
    }
    if (bad) {
        if (err_line) *err_line = bad;
        return fail(TIO_ERR_INVALID, "line %lld not in the fast format", (long long)bad);
    }
    tio_parsed_trace *r = new tio_parsed_trace();
    r->meta = meta;
    std::unordered_map<std::string, int32_t> code;
    for (auto &pt : parts) {
        for (size_t i = 0; i < pt.k_dur.size(); ++i) {
            r->k_index.push_back(pt.k_index[i]); r->k_dur.push_back(pt.k_dur[i]);
            r->k_stage.push_back(pt.k_stage[i]); r->k_layer.push_back(pt.k_layer[i]);
            const std::string key = (pt.k_name_esc[i] ? "\x01" : "") + pt.k_name[i];
            auto it = code.find(key);
            int32_t cd;
            if (it == code.end()) {
                cd = (int32_t)r->name_off.size();
                code.emplace(key, cd);
                r->name_off.push_back((int64_t)r->names.size());
                r->names += pt.k_name[i];
                r->name_esc.push_back(pt.k_name_esc[i]);
            } else {
                cd = it->second;
            }
            r->k_code.push_back(cd);
        }
    }
    r->name_off.push_back((int64_t)r->names.size());
    r->ptr.push_back(0);
    for (auto &pt : parts) {
        r->t_id.insert(r->t_id.end(), pt.t_id.begin(), pt.t_id.end());
        r->t_size.insert(r->t_size.end(), pt.t_size.begin(), pt.t_size.end());
        r->t_kind.insert(r->t_kind.end(), pt.t_kind.begin(), pt.t_kind.end());
        r->t_layer.insert(r->t_layer.end(), pt.t_layer.begin(), pt.t_layer.end());
        for (int64_t c : pt.t_count) r->ptr.push_back(r->ptr.back() + c);
        r->acc.insert(r->acc.end(), pt.acc.begin(), pt.acc.end());
    }
    *out = r;
    return TIO_OK;
}

extern "C" int tio_parsed_sizes(const tio_parsed_trace *r, int64_t *n_kernels, int64_t *n_tensors,
                                int64_t *n_events, int64_t *n_names, int64_t *names_bytes, int64_t *meta_bytes) {
    if (!r) return fail(TIO_ERR_INVALID, "null parsed trace");
    *n_kernels = (int64_t)r->k_dur.size();
    *n_tensors = (int64_t)r->t_id.size();
    *n_events = (int64_t)r->acc.size();
    *n_names = (int64_t)r->name_esc.size();
    *names_bytes = (int64_t)r->names.size();
    *meta_bytes = (int64_t)r->meta.size();
    return TIO_OK;
}

extern "C" int tio_parsed_copy(const tio_parsed_trace *r, int64_t *k_index, int64_t *k_dur, int32_t *k_code,
                               int64_t *k_stage, int64_t *k_layer, int64_t *t_id, int64_t *t_size, int8_t *t_kind,
                               int64_t *t_layer, int64_t *ptr, int64_t *acc, char *names, int64_t *name_off,
                               uint8_t *name_esc, char *meta) {
    if (!r) return fail(TIO_ERR_INVALID, "null parsed trace");
    auto cp = [](void *dst, const void *src, size_t n) { if (dst && n) memcpy(dst, src, n); };
    const size_t N = r->k_dur.size(), T = r->t_id.size();
    cp(k_index, r->k_index.data(), 8 * N); cp(k_dur, r->k_dur.data(), 8 * N); cp(k_code, r->k_code.data(), 4 * N);
    cp(k_stage, r->k_stage.data(), 8 * N); cp(k_layer, r->k_layer.data(), 8 * N);
    cp(t_id, r->t_id.data(), 8 * T); cp(t_size, r->t_size.data(), 8 * T); cp(t_kind, r->t_kind.data(), T);
    cp(t_layer, r->t_layer.data(), 8 * T); cp(ptr, r->ptr.data(), 8 * (T + 1)); cp(acc, r->acc.data(), 8 * r->acc.size());
    cp(names, r->names.data(), r->names.size()); cp(name_off, r->name_off.data(), 8 * r->name_off.size());
    cp(name_esc, r->name_esc.data(), r->name_esc.size()); cp(meta, r->meta.data(), r->meta.size());
    return TIO_OK;
}

extern "C" int tio_parsed_destroy(tio_parsed_trace *r) {
    delete r;
    return TIO_OK;
}
