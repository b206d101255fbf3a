// Native NDJSON trace ingest: the reference's parse_trace
// (traceio.py:153-191, wire format traceio.py:1-23) reads ~0.07 M events/s in Python.
// This parser splits the input at line boundaries over host threads and turns every
// well-formed record straight into SoA columns plus a deduplicated location table.
// It accepts exactly the records the reference accepts without error and lists every line
// it cannot vouch for (any JSON or field-rule irregularity, up to 64k per chunk) without
// returning columns; the Python layer checks just those lines the reference's way --
// raising its exact exception for the first bad one, or rewriting an unusual-but-valid
// line in canonical form -- and calls the parser again on the patched input.  Sorting by
// (t0, seq) and validation run on the GPU afterwards.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "b2l.h"

namespace b2l {
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

namespace ingest {

struct Loc {
    uint64_t codeptr;
    int64_t line;  // -1 = None
    bool has_file;
    std::string file;
    bool operator==(const Loc &o) const {
        return codeptr == o.codeptr && line == o.line && has_file == o.has_file && file == o.file;
    }
};
struct LocHash {
    size_t operator()(const Loc &l) const {
        return std::hash<std::string>()(l.file) ^ (l.codeptr * 0x9E3779B97F4A7C15ull) ^ (size_t)(l.line * 31) ^
               (l.has_file ? 0x55 : 0);
    }
};

struct Chunk {
    std::vector<uint64_t> c[9];  // seq t0 t1 src dst src_addr dst_addr bytes hash
    std::vector<uint8_t> kind;
    std::vector<uint32_t> loc;   // chunk-local loc ids
    std::vector<Loc> locs;
    std::unordered_map<Loc, uint32_t, LocHash> loc_ids;
    std::vector<uint64_t> err_lines;  // lines the parser cannot vouch for (1-based, ascending)
};
constexpr size_t MAX_ERR_LINES = size_t(1) << 16;  // per chunk and call; the caller re-parses after patching

// ------------------------------------------------------------------ a strict JSON scanner
struct Scan {
    const char *p, *e;
    bool ok = true;
    void ws() {
        while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool lit(const char *s) {
        size_t n = strlen(s);
        if ((size_t)(e - p) < n || memcmp(p, s, n) != 0) return false;
        p += n;
        return true;
    }
    static void put_utf8(std::string &o, uint32_t cp) {
        if (cp < 0x80) {
            o += (char)cp;
        } else if (cp < 0x800) {
            o += (char)(0xC0 | (cp >> 6)), o += (char)(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += (char)(0xE0 | (cp >> 12)), o += (char)(0x80 | ((cp >> 6) & 0x3F)), o += (char)(0x80 | (cp & 0x3F));
        } else {
            o += (char)(0xF0 | (cp >> 18)), o += (char)(0x80 | ((cp >> 12) & 0x3F));
            o += (char)(0x80 | ((cp >> 6) & 0x3F)), o += (char)(0x80 | (cp & 0x3F));
        }
    }
    bool hex4(uint32_t &v) {
        if (e - p < 4) return false;
        v = 0;
        for (int i = 0; i < 4; ++i) {
            char ch = p[i];
            v <<= 4;
            if (ch >= '0' && ch <= '9') v |= (uint32_t)(ch - '0');
            else if (ch >= 'a' && ch <= 'f') v |= (uint32_t)(ch - 'a' + 10);
            else if (ch >= 'A' && ch <= 'F') v |= (uint32_t)(ch - 'A' + 10);
            else return false;
        }
        p += 4;
        return true;
    }
    // JSON string (after the opening quote is consumed by the caller)
    bool str(std::string &o) {
        o.clear();
        while (p < e) {
            unsigned char ch = (unsigned char)*p++;
            if (ch == '"') return true;
            if (ch < 0x20) return false;  // Python's json rejects raw control characters
            if (ch != '\\') {
                o += (char)ch;
                continue;
            }
            if (p >= e) return false;
            char esc = *p++;
            switch (esc) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    uint32_t v;
                    if (!hex4(v)) return false;
                    if (v >= 0xD800 && v < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
                        // a surrogate pair combines as Python's json does; anything else after a
                        // high surrogate leaves it lone (and is read as its own escape next)
                        const char *save = p;
                        uint32_t lo;
                        p += 2;
                        if (hex4(lo) && lo >= 0xDC00 && lo < 0xE000) v = 0x10000 + ((v - 0xD800) << 10) + (lo - 0xDC00);
                        else p = save;
                    }
                    // lone surrogates are kept as their 3-byte form (Python decodes the names
                    // with "surrogatepass"), NULs as a 0 byte: names carry explicit lengths
                    put_utf8(o, v);
                    break;
                }
                default: return false;
            }
        }
        return false;
    }
    // value kinds
    enum { V_UINT, V_STR, V_NULL, V_OTHER };
    // Parse any JSON value; integers must be plain non-negative u64 literals to count as V_UINT.
    int value(uint64_t &u, std::string &s) {
        ws();
        if (p >= e) return -1;
        char ch = *p;
        if (ch == '"') {
            ++p;
            return str(s) ? V_STR : -1;
        }
        if (ch == 'n') return lit("null") ? V_NULL : -1;
        if (ch == 't') return lit("true") ? V_OTHER : -1;
        if (ch == 'f') return lit("false") ? V_OTHER : -1;
        if (ch == '{' || ch == '[') return skip_container() ? V_OTHER : -1;
        if (ch == '-' || (ch >= '0' && ch <= '9')) {
            bool neg = false, frac = false, over = false;
            uint64_t v = 0;
            if (!number(neg, frac, over, v)) return -1;
            if (frac || neg || over) return -2;  // a float / negative / > u64: the reference rejects it
            u = v;
            return V_UINT;
        }
        return -1;
    }
    // JSON number grammar: -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)?
    bool number(bool &neg, bool &frac, bool &over, uint64_t &v) {
        if (p < e && *p == '-') neg = true, ++p;
        if (p >= e || *p < '0' || *p > '9') return false;
        if (*p == '0') {
            ++p;
        } else {
            while (p < e && *p >= '0' && *p <= '9') {
                const uint64_t d = (uint64_t)(*p - '0');
                if (v > (UINT64_MAX - d) / 10) over = true;
                v = v * 10 + d;
                ++p;
            }
        }
        if (p < e && *p == '.') {
            frac = true, ++p;
            if (p >= e || *p < '0' || *p > '9') return false;
            while (p < e && *p >= '0' && *p <= '9') ++p;
        }
        if (p < e && (*p == 'e' || *p == 'E')) {
            frac = true, ++p;
            if (p < e && (*p == '+' || *p == '-')) ++p;
            if (p >= e || *p < '0' || *p > '9') return false;
            while (p < e && *p >= '0' && *p <= '9') ++p;
        }
        return true;
    }
    // strict skip of one nested object/array (valid JSON only; depth-limited)
    bool skip_container(int depth = 0) {
        if (depth > 64) return false;
        std::string tmp;
        const char open = *p++;
        const char close = open == '{' ? '}' : ']';
        ws();
        if (p < e && *p == close) {
            ++p;
            return true;
        }
        for (;;) {
            ws();
            if (open == '{') {
                if (p >= e || *p != '"') return false;
                ++p;
                if (!str(tmp)) return false;
                ws();
                if (p >= e || *p != ':') return false;
                ++p;
            }
            ws();
            if (p >= e) return false;
            const char ch = *p;
            if (ch == '{' || ch == '[') {
                if (!skip_container(depth + 1)) return false;
            } else {
                uint64_t u = 0;
                int t = value(u, tmp);
                if (t == -1) return false;
            }
            ws();
            if (p < e && *p == ',') {
                ++p;
                continue;
            }
            if (p < e && *p == close) {
                ++p;
                return true;
            }
            return false;
        }
    }
};

enum : uint32_t {
    F_SEQ = 1 << 0, F_KIND = 1 << 1, F_T0 = 1 << 2, F_T1 = 1 << 3, F_SRC = 1 << 4, F_DST = 1 << 5,
    F_SA = 1 << 6, F_DA = 1 << 7, F_BYTES = 1 << 8, F_HASH = 1 << 9, F_CODEPTR = 1 << 10, F_REQUIRED = (1 << 11) - 1
};

// One event record -> values; false = the fast path cannot vouch for this line.
bool parse_event(const char *b, const char *e, uint64_t v[9], uint8_t &kind, Loc &loc) {
    Scan sc{b, e};
    sc.ws();
    if (sc.p >= sc.e || *sc.p != '{') return false;
    ++sc.p;
    uint32_t have = 0;
    bool file_present = false, line_present = false, file_is_str = false, line_ok = false;
    std::string key, sval, file;
    uint64_t u = 0, line = 0;
    sc.ws();
    if (sc.p < sc.e && *sc.p == '}') {
        ++sc.p;
    } else {
        for (;;) {
            sc.ws();
            if (sc.p >= sc.e || *sc.p != '"') return false;
            ++sc.p;
            if (!sc.str(key)) return false;
            sc.ws();
            if (sc.p >= sc.e || *sc.p != ':') return false;
            ++sc.p;
            int t = sc.value(u, sval);
            if (t == -1) return false;
            auto need_uint = [&](uint32_t bit, int slot) {
                if (t != Scan::V_UINT) return false;
                have |= bit;
                v[slot] = u;
                return true;
            };
            if (key == "seq") { if (!need_uint(F_SEQ, 0)) return false; }
            else if (key == "t0") { if (!need_uint(F_T0, 1)) return false; }
            else if (key == "t1") { if (!need_uint(F_T1, 2)) return false; }
            else if (key == "src_dev") { if (!need_uint(F_SRC, 3)) return false; }
            else if (key == "dst_dev") { if (!need_uint(F_DST, 4)) return false; }
            else if (key == "src_addr") { if (!need_uint(F_SA, 5)) return false; }
            else if (key == "dst_addr") { if (!need_uint(F_DA, 6)) return false; }
            else if (key == "bytes") { if (!need_uint(F_BYTES, 7)) return false; }
            else if (key == "hash") { if (!need_uint(F_HASH, 8)) return false; }
            else if (key == "codeptr") {
                if (t != Scan::V_UINT) return false;
                have |= F_CODEPTR;
                loc.codeptr = u;
            } else if (key == "kind") {
                if (t != Scan::V_STR) return false;
                have |= F_KIND;
                if (sval == "transfer") kind = B2L_KIND_TRANSFER;
                else if (sval == "alloc") kind = B2L_KIND_ALLOC;
                else if (sval == "delete") kind = B2L_KIND_DELETE;
                else if (sval == "kernel") kind = B2L_KIND_KERNEL;
                else return false;
            } else if (key == "file") {
                if (t == Scan::V_NULL) file_present = false, file_is_str = false;
                else if (t == Scan::V_STR) file_present = true, file_is_str = true, file = sval;
                else return false;
            } else if (key == "line") {
                if (t == Scan::V_NULL) line_present = false, line_ok = false;
                else if (t == Scan::V_UINT && u > 0 && u <= (uint64_t)INT64_MAX) line_present = true, line_ok = true,
                                                                                   line = u;
                else return false;
            } else if (t == -2) {
                // an unknown field with an out-of-range number is still valid JSON: accept
            }
            sc.ws();
            if (sc.p < sc.e && *sc.p == ',') {
                ++sc.p;
                continue;
            }
            if (sc.p < sc.e && *sc.p == '}') {
                ++sc.p;
                break;
            }
            return false;
        }
    }
    sc.ws();
    if (sc.p != sc.e) return false;  // trailing data: invalid JSON
    if ((have & F_REQUIRED) != F_REQUIRED) return false;
    if (v[2] < v[1]) return false;   // inverted interval
    if (file_present && !line_present) return false;
    (void)file_is_str;
    (void)line_ok;
    loc.has_file = file_present;
    loc.file = file_present ? file : std::string();
    loc.line = line_present ? (int64_t)line : -1;
    return true;
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// ------------------------------------------------------------------ canonical-line fast path
// The capture agents write one shape (model.ts:38-48 serializeEvent, b2l_capture.cu): the eleven
// fields in wire order, no whitespace, plain integers, optionally ,"file":"...","line":N.  Such
// a line is decoded with fixed literals and digit loops (no allocation); anything else -- other
// key orders, whitespace, escapes, leading zeros, u64 overflow, unknown fields -- returns false
// and the general scanner decides, so accepted lines give exactly the general parser's result.
struct Fast {
    const char *p, *e;
    bool lit(const char *s, size_t n) {
        if ((size_t)(e - p) < n || memcmp(p, s, n) != 0) return false;
        p += n;
        return true;
    }
    bool uint(uint64_t &v) {  // JSON non-negative integer without leading zeros, no overflow
        if (p >= e || *p < '0' || *p > '9') return false;
        if (*p == '0') {
            ++p;
            v = 0;
            return p >= e || *p < '0' || *p > '9';
        }
        uint64_t x = 0;
        int nd = 0;
        while (p < e && *p >= '0' && *p <= '9') {
            if (++nd > 19) return false;  // 20 digits may overflow: the general path checks
            x = x * 10 + (uint64_t)(*p++ - '0');
        }
        if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) return false;
        v = x;
        return true;
    }
};
#define FLIT(s) f.lit(s, sizeof(s) - 1)
bool parse_event_fast(const char *b, const char *e, uint64_t v[9], uint8_t &kind, uint64_t &codeptr,
                      const char *&file, size_t &file_len, uint64_t &line) {
    Fast f{b, e};
    if (!FLIT("{\"seq\":") || !f.uint(v[0]) || !FLIT(",\"kind\":\"")) return false;
    if (FLIT("transfer\"")) kind = B2L_KIND_TRANSFER;
    else if (FLIT("alloc\"")) kind = B2L_KIND_ALLOC;
    else if (FLIT("delete\"")) kind = B2L_KIND_DELETE;
    else if (FLIT("kernel\"")) kind = B2L_KIND_KERNEL;
    else return false;
    if (!FLIT(",\"t0\":") || !f.uint(v[1]) || !FLIT(",\"t1\":") || !f.uint(v[2])) return false;
    if (!FLIT(",\"src_dev\":") || !f.uint(v[3]) || !FLIT(",\"dst_dev\":") || !f.uint(v[4])) return false;
    if (!FLIT(",\"src_addr\":") || !f.uint(v[5]) || !FLIT(",\"dst_addr\":") || !f.uint(v[6])) return false;
    if (!FLIT(",\"bytes\":") || !f.uint(v[7]) || !FLIT(",\"hash\":") || !f.uint(v[8])) return false;
    if (!FLIT(",\"codeptr\":") || !f.uint(codeptr)) return false;
    file = nullptr, file_len = 0, line = 0;
    if (f.p < f.e && *f.p == ',') {
        if (!FLIT(",\"file\":\"")) return false;
        const char *s0 = f.p;
        while (f.p < f.e && *f.p != '"') {
            const unsigned char ch = (unsigned char)*f.p;
            if (ch < 0x20 || ch == '\\' || ch >= 0x80) return false;  // escapes / control / non-ASCII: general path
            ++f.p;
        }
        if (f.p >= f.e) return false;
        file = s0, file_len = (size_t)(f.p - s0);
        ++f.p;
        if (!FLIT(",\"line\":") || !f.uint(line) || line == 0 || line > (uint64_t)INT64_MAX) return false;
    }
    if (!FLIT("}") || f.p != f.e) return false;
    return v[2] >= v[1];  // an inverted interval is the general path's (and the reference's) error
}
#undef FLIT

void parse_range(const char *data, size_t lo, size_t hi, uint64_t first_line, Chunk &ck) {
    uint64_t line_no = first_line;
    size_t i = lo;
    uint64_t v[9];
    static const bool use_fast = getenv("B2L_INGEST_GENERAL_ONLY") == nullptr;  // tests compare both paths
    const size_t guess = (hi - lo) / 128 + 16;  // capture-agent lines are ~150-180 bytes
    for (int k = 0; k < 9; ++k) ck.c[k].reserve(guess);
    ck.kind.reserve(guess);
    ck.loc.reserve(guess);
    // location ids of codeptr-only locations (the common case): a small direct-mapped cache in
    // front of the general table
    constexpr int LC = 64;
    uint64_t lc_key[LC];
    uint32_t lc_id[LC];
    bool lc_ok[LC] = {false};
    auto loc_id = [&](const Loc &loc) {
        auto it = ck.loc_ids.find(loc);
        if (it != ck.loc_ids.end()) return it->second;
        const uint32_t id = (uint32_t)ck.locs.size();
        ck.loc_ids.emplace(loc, id);
        ck.locs.push_back(loc);
        return id;
    };
    while (i < hi) {
        const char *nl = (const char *)memchr(data + i, '\n', hi - i);
        const size_t j = nl ? (size_t)(nl - data) : hi;
        const char *b = data + i, *e = data + j;
        while (b < e && is_ws(*b)) ++b;
        while (e > b && is_ws(e[-1])) --e;
        if (b < e && *b != '#') {
            uint8_t kind = 0;
            uint64_t codeptr = 0, line = 0;
            const char *file = nullptr;
            size_t flen = 0;
            uint32_t id;
            if (use_fast && parse_event_fast(b, e, v, kind, codeptr, file, flen, line)) {
                if (!file) {
                    const int h = (int)((codeptr * 0x9E3779B97F4A7C15ull) >> 58);
                    if (lc_ok[h] && lc_key[h] == codeptr) {
                        id = lc_id[h];
                    } else {
                        id = loc_id(Loc{codeptr, -1, false, std::string()});
                        lc_ok[h] = true, lc_key[h] = codeptr, lc_id[h] = id;
                    }
                } else {
                    id = loc_id(Loc{codeptr, (int64_t)line, true, std::string(file, flen)});
                }
            } else {
                Loc loc{0, -1, false, std::string()};
                if (!parse_event(b, e, v, kind, loc)) {
                    ck.err_lines.push_back(line_no);
                    if (ck.err_lines.size() >= MAX_ERR_LINES) return;
                    i = j + 1;
                    ++line_no;
                    continue;
                }
                id = loc_id(loc);
            }
            for (int k = 0; k < 9; ++k) ck.c[k].push_back(v[k]);
            ck.kind.push_back(kind);
            ck.loc.push_back(id);
        }
        i = j + 1;
        ++line_no;
    }
}

}  // namespace ingest
}  // namespace b2l

// ------------------------------------------------------------------------ C ABI
struct b2l_ingest_impl {
    b2l_ingest pub;
    std::vector<uint64_t> cols[9];
    std::vector<uint8_t> kind;
    std::vector<uint32_t> loc;
    std::vector<uint64_t> loc_codeptr;
    std::vector<int64_t> loc_line;
    std::vector<uint64_t> loc_file_off;
    std::vector<uint32_t> loc_file_len;
    std::string strings;
    std::vector<uint64_t> err_lines;
};

extern "C" {

int b2l_ingest_ndjson(const char *data, uint64_t len, int threads, b2l_ingest **out) {
    using namespace b2l::ingest;
    if (!out || (len && !data)) return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    auto *R = new b2l_ingest_impl();
    memset(&R->pub, 0, sizeof(R->pub));
    *out = &R->pub;
    // ---- header: the first non-blank, non-comment line
    size_t i = 0;
    uint64_t line_no = 1;
    bool found = false;
    size_t body = len;
    while (i < len) {
        size_t j = i;
        while (j < len && data[j] != '\n') ++j;
        const char *b = data + i, *e = data + j;
        while (b < e && is_ws(*b)) ++b;
        while (e > b && is_ws(e[-1])) --e;
        if (b < e && *b != '#') {
            found = true;
            R->pub.header_line = line_no;
            // header fields (all must be plain u64 literals; anything else -> the Python path)
            Scan sc{b, e};
            bool ok = true, have_v = false, have_nd = false, have_h = false;
            std::string key, sval;
            uint64_t u = 0;
            sc.ws();
            if (sc.p >= sc.e || *sc.p != '{') ok = false;
            else ++sc.p;
            sc.ws();
            if (ok && sc.p < sc.e && *sc.p == '}') {
                ++sc.p;
            } else {
                while (ok) {
                    sc.ws();
                    if (sc.p >= sc.e || *sc.p != '"') { ok = false; break; }
                    ++sc.p;
                    if (!sc.str(key)) { ok = false; break; }
                    sc.ws();
                    if (sc.p >= sc.e || *sc.p != ':') { ok = false; break; }
                    ++sc.p;
                    int t = sc.value(u, sval);
                    if (t == -1) { ok = false; break; }
                    if (key == "dmlens") { if (t != Scan::V_UINT) ok = false; R->pub.version = u, have_v = true; }
                    else if (key == "num_devices") { if (t != Scan::V_UINT) ok = false; R->pub.num_devices = u, have_nd = true; }
                    else if (key == "host_device") { if (t != Scan::V_UINT) ok = false; R->pub.host_device = u, have_h = true; }
                    else if (key == "wall_time_ns") { if (t != Scan::V_UINT) ok = false; R->pub.wall_time_ns = u, R->pub.has_wall = 1; }
                    sc.ws();
                    if (sc.p < sc.e && *sc.p == ',') { ++sc.p; continue; }
                    if (sc.p < sc.e && *sc.p == '}') { ++sc.p; break; }
                    ok = false;
                }
            }
            sc.ws();
            if (sc.p != sc.e) ok = false;
            if (!ok || !have_v || R->pub.version != 1 || !have_nd || !have_h) {
                R->pub.err_line = line_no;
                R->err_lines.push_back(line_no);
                R->pub.n_err_lines = 1;
                R->pub.err_lines = R->err_lines.data();
                return B2L_OK;
            }
            body = j + 1 <= len ? j + 1 : len;
            ++line_no;
            break;
        }
        i = j + 1;
        ++line_no;
    }
    if (!found) {
        R->pub.err_line = line_no;  // MissingHeader: the Python path names it
        R->pub.header_line = 0;
        return B2L_OK;
    }
    // ---- events: split the body at line starts across threads
    if (threads < 1) threads = 1;
    size_t rest = len > body ? len - body : 0;
    int T = (int)std::min<size_t>((size_t)threads, std::max<size_t>(1, rest / (1 << 20)));
    std::vector<size_t> cut(T + 1);
    cut[0] = body;
    cut[T] = len;
    for (int t = 1; t < T; ++t) {
        size_t c = body + rest * t / T;
        while (c < len && data[c - 1] != '\n') ++c;
        cut[t] = std::max(c, cut[t - 1]);
    }
    std::vector<uint64_t> first(T);
    first[0] = line_no;
    {
        std::vector<uint64_t> nl(T, 0);
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] { nl[t] = (uint64_t)std::count(data + cut[t], data + cut[t + 1], '\n'); });
        for (auto &x : th) x.join();
        for (int t = 1; t < T; ++t) first[t] = first[t - 1] + nl[t - 1];
    }
    std::vector<Chunk> ck(T);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back([&, t] { parse_range(data, cut[t], cut[t + 1], first[t], ck[t]); });
        for (auto &x : th) x.join();
    }
    for (int t = 0; t < T; ++t) {  // a chunk that stopped at the cap ends the list: nothing after it was read
        R->err_lines.insert(R->err_lines.end(), ck[t].err_lines.begin(), ck[t].err_lines.end());
        if (ck[t].err_lines.size() >= MAX_ERR_LINES) break;
    }
    if (!R->err_lines.empty()) {
        R->pub.err_line = R->err_lines[0];
        R->pub.n_err_lines = R->err_lines.size();
        R->pub.err_lines = R->err_lines.data();
        return B2L_OK;
    }
    // ---- merge chunks; global location ids
    size_t n = 0;
    for (auto &c : ck) n += c.kind.size();
    for (int k = 0; k < 9; ++k) R->cols[k].reserve(n);
    R->kind.reserve(n);
    R->loc.reserve(n);
    std::unordered_map<Loc, uint32_t, LocHash> gids;
    for (auto &c : ck) {
        std::vector<uint32_t> remap(c.locs.size());
        for (size_t l = 0; l < c.locs.size(); ++l) {
            auto it = gids.find(c.locs[l]);
            if (it == gids.end()) {
                uint32_t id = (uint32_t)R->loc_codeptr.size();
                gids.emplace(c.locs[l], id);
                R->loc_codeptr.push_back(c.locs[l].codeptr);
                R->loc_line.push_back(c.locs[l].line);
                if (c.locs[l].has_file) {
                    R->loc_file_off.push_back(R->strings.size());
                    R->loc_file_len.push_back((uint32_t)c.locs[l].file.size());
                    R->strings += c.locs[l].file;
                } else {
                    R->loc_file_off.push_back(UINT64_MAX);
                    R->loc_file_len.push_back(0);
                }
                remap[l] = id;
            } else {
                remap[l] = it->second;
            }
        }
        for (int k = 0; k < 9; ++k) R->cols[k].insert(R->cols[k].end(), c.c[k].begin(), c.c[k].end());
        R->kind.insert(R->kind.end(), c.kind.begin(), c.kind.end());
        for (uint32_t id : c.loc) R->loc.push_back(remap[id]);
    }
    b2l_ingest &P = R->pub;
    P.n_events = n;
    P.seq = R->cols[0].data(), P.start_ns = R->cols[1].data(), P.end_ns = R->cols[2].data();
    P.src_device = R->cols[3].data(), P.dst_device = R->cols[4].data(), P.src_addr = R->cols[5].data();
    P.dst_addr = R->cols[6].data(), P.bytes = R->cols[7].data(), P.hash = R->cols[8].data();
    P.kind = R->kind.data(), P.loc = R->loc.data();
    P.n_locs = (uint32_t)R->loc_codeptr.size();
    P.loc_codeptr = R->loc_codeptr.data(), P.loc_line = R->loc_line.data();
    P.loc_file_off = R->loc_file_off.data(), P.loc_file_len = R->loc_file_len.data();
    P.strings = R->strings.data();
    return B2L_OK;
}

void b2l_ingest_free(b2l_ingest *p) {
    if (!p) return;
    delete reinterpret_cast<b2l_ingest_impl *>(p);  // pub is the first member
}

// serialize_trace's body (traceio.py:193-237): every event as one canonical line, in the given
// order, over host threads: lengths per chunk first, then each chunk writes its own slice.
int b2l_serialize_ndjson(const b2l_trace_cols *c, const char *header, uint64_t header_len, const char *suffix_data,
                         const uint64_t *suffix_off, int threads, char **text, uint64_t *len) {
    if (!c || !text || !len || (header_len && !header) || (c->n_locs && (!suffix_data || !suffix_off)))
        return b2l::fail(B2L_E_INVALID_ARG, "null argument");
    if (c->device_resident) return b2l::fail(B2L_E_INVALID_ARG, "b2l_serialize_ndjson needs host columns");
    const uint64_t n = c->n_events;
    for (uint64_t i = 0; i < n; ++i)
        if (c->loc[i] >= c->n_locs || c->kind[i] > 3) return b2l::fail(B2L_E_INVALID_ARG, "bad kind or location id");
    static const char *kname[4] = {"transfer", "alloc", "delete", "kernel"};
    // one event line; writes at most 11 keys + 9 u64 + 2 i32 + the suffix
    auto line = [&](uint64_t i, char *o) -> size_t {
        char *p = o;
        auto lit = [&](const char *s, size_t k) { memcpy(p, s, k), p += k; };
        auto u = [&](uint64_t v) { p = std::to_chars(p, p + 20, v).ptr; };
        auto d = [&](int32_t v) { p = std::to_chars(p, p + 11, v).ptr; };
        lit("{\"seq\":", 7), u(c->seq[i]);
        lit(",\"kind\":\"", 9);
        const char *k = kname[c->kind[i]];
        lit(k, strlen(k));
        lit("\",\"t0\":", 7), u(c->start_ns[i]);
        lit(",\"t1\":", 6), u(c->end_ns[i]);
        lit(",\"src_dev\":", 11), d(c->src_device[i]);
        lit(",\"dst_dev\":", 11), d(c->dst_device[i]);
        lit(",\"src_addr\":", 12), u(c->src_addr[i]);
        lit(",\"dst_addr\":", 12), u(c->dst_addr[i]);
        lit(",\"bytes\":", 9), u(c->bytes[i]);
        lit(",\"hash\":", 8), u(c->hash[i]);
        const uint32_t l = c->loc[i];
        lit(suffix_data + suffix_off[l], suffix_off[l + 1] - suffix_off[l]);  // ,"codeptr":..[,"file":..,"line":..]}
        *p++ = '\n';
        return (size_t)(p - o);
    };
    uint64_t max_suffix = 0;
    for (uint32_t l = 0; l < c->n_locs; ++l) max_suffix = std::max(max_suffix, suffix_off[l + 1] - suffix_off[l]);
    const size_t bound = 256 + max_suffix;  // per line
    if (threads < 1) threads = 1;
    const int T = (int)std::min<uint64_t>((uint64_t)threads, std::max<uint64_t>(1, n / 65536));
    std::vector<uint64_t> lo(T + 1);
    for (int t = 0; t <= T; ++t) lo[t] = n * (uint64_t)t / (uint64_t)T;
    std::vector<std::string> part(T);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                std::string &o = part[t];
                o.resize((size_t)(lo[t + 1] - lo[t]) * 160 + bound);
                size_t w = 0;
                for (uint64_t i = lo[t]; i < lo[t + 1]; ++i) {
                    if (o.size() - w < bound) o.resize(o.size() * 2 + bound);
                    w += line(i, &o[w]);
                }
                o.resize(w);
            });
        for (auto &x : th) x.join();
    }
    size_t total = header_len;
    for (auto &p : part) total += p.size();
    char *out = (char *)malloc(total + 1);
    if (!out) return b2l::fail(B2L_E_OOM, "host allocation failed");
    memcpy(out, header, header_len);
    size_t w = header_len;
    for (auto &p : part) memcpy(out + w, p.data(), p.size()), w += p.size();
    out[total] = 0;
    *text = out;
    *len = total;
    return B2L_OK;
}

void b2l_serialize_free(char *text) { free(text); }

}  // extern "C"
