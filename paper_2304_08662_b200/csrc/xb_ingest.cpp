// Ingest of the reference's input formats straight into contiguous buffers
// (SURVEY §8(f) item 2): FASTA records -> one symbol buffer + offsets (then
// xb_pool_add_bulk packs them), seed lists and Matrix Market overlaps ->
// xb_task arrays.  Semantics are the reference parsers' (proj/src/io.cpp):
// line splitting (for_lines, io.cpp:17-30), tokenising (split_ws, 32-43),
// integer fields (parse_ll = std::stoll over the whole token, 45-54), the
// error taxonomy (errors.hpp:54-82) with the same kind, line and message.
// FASTA is parsed by all host threads over chunks cut at "\n>" boundaries;
// errors are resolved in line order, so results equal a sequential parse.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../../include/xdrop_b200.h"

namespace {

struct ParseFail {
    int kind = XB_PARSE_OK;
    int64_t line = 0;
    std::string msg;
};

void set_err(xb_parse_error* e, const ParseFail& f) {
    if (!e) return;
    e->kind = f.kind;
    e->reserved = 0;
    e->line = f.line;
    const size_t n = std::min(f.msg.size(), sizeof(e->message) - 1);
    std::memcpy(e->message, f.msg.data(), n);
    e->message[n] = 0;
}

void clear_err(xb_parse_error* e) {
    if (!e) return;
    e->kind = XB_PARSE_OK;
    e->reserved = 0;
    e->line = 0;
    e->message[0] = 0;
}

inline bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// for_lines (io.cpp:17-30): LF or CRLF lines, 1-based numbers, the text
// after the last LF is a line too.  fn returns false to stop.
template <typename F>
void for_lines(std::string_view text, int64_t first_line, F&& fn) {
    size_t pos = 0;
    int64_t line = first_line - 1;
    while (pos <= text.size()) {
        const void* hit = std::memchr(text.data() + pos, '\n', text.size() - pos);
        const size_t nl = hit ? size_t(static_cast<const char*>(hit) - text.data()) : std::string_view::npos;
        const size_t end = nl == std::string_view::npos ? text.size() : nl;
        size_t len = end - pos;
        if (len > 0 && text[pos + len - 1] == '\r') --len;
        ++line;
        if (!fn(text.substr(pos, len), line)) return;
        if (nl == std::string_view::npos) break;
        pos = nl + 1;
    }
}

// split_ws (io.cpp:32-43)
void split_ws(std::string_view s, std::vector<std::string_view>& out) {
    out.clear();
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && is_space(s[i])) ++i;
        size_t j = i;
        while (j < s.size() && !is_space(s[j])) ++j;
        if (j > i) out.push_back(s.substr(i, j - i));
        i = j;
    }
}

// parse_ll (io.cpp:45-54): std::stoll must consume the whole token.  stoll
// is strtoll in base 10: an optional sign ('+' too), digits; out of range
// throws (-> not an integer).  Tokens never hold whitespace (split_ws).
bool parse_ll(std::string_view tok, long long& out) {
    if (tok.empty()) return false;
    const char* b = tok.data();
    const char* e = tok.data() + tok.size();
    if (*b == '+') {  // from_chars takes '-' but not '+'
        ++b;
        if (b == e || *b == '-' || *b == '+') return false;
    }
    long long v = 0;
    const auto r = std::from_chars(b, e, v, 10);
    if (r.ec != std::errc() || r.ptr != e) return false;
    out = v;
    return true;
}

std::string L(int64_t n) { return std::to_string(n); }

// ---------------------------------------------------------------- FASTA --

struct FastaChunk {
    std::string_view text;
    int64_t first_line = 1;
    // output
    std::vector<char> sym;
    std::vector<int64_t> rec_end;    // end offset (in sym) of each record
    std::vector<std::string> names;
    ParseFail fail;                  // first error inside the chunk
    bool last_empty = false;         // its last record has no data (io.cpp:66-68, 91-92)
};

constexpr uint8_t kSkip = 0xFE, kBad = 0xFF;

// per byte: isspace -> kSkip; else toupper, kBad unless allowed (io.cpp:81-89)
void fasta_classes(const char* allowed, uint8_t (&cls)[256]) {
    bool valid[256] = {};
    for (const char* a = allowed; *a; ++a)
        valid[static_cast<unsigned char>(std::toupper(static_cast<unsigned char>(*a)))] = true;
    for (int c = 0; c < 256; ++c) {
        const unsigned char u = static_cast<unsigned char>(std::toupper(c));
        cls[c] = std::isspace(c) ? kSkip : (valid[u] && u < kSkip ? u : kBad);
    }
}

void parse_fasta_chunk(FastaChunk& C, const uint8_t (&cls)[256]) {
    bool have = false;
    int64_t rec_start = 0;
    for_lines(C.text, C.first_line, [&](std::string_view line, int64_t lineno) {
        if (line.empty()) return true;
        if (line[0] == '>') {
            if (have && int64_t(C.sym.size()) == rec_start) {
                C.fail = {XB_PARSE_EMPTY_RECORD, 0,
                          "record '" + C.names.back() + "' has no sequence data"};
                return false;
            }
            if (have) C.rec_end.push_back(int64_t(C.sym.size()));
            std::string_view rest = line.substr(1);
            size_t i = 0;
            while (i < rest.size() && is_space(rest[i])) ++i;
            size_t j = i;
            while (j < rest.size() && !is_space(rest[j])) ++j;
            C.names.emplace_back(rest.substr(i, j - i));
            rec_start = int64_t(C.sym.size());
            have = true;
            return true;
        }
        if (!have) {  // only possible before the first header of the text
            C.fail = {XB_PARSE_MISSING_HEADER, 0,
                      "sequence data on line " + L(lineno) + " appears before any '>' header"};
            return false;
        }
        // class table: the upper-cased symbol, kSkip (whitespace) or kBad
        const size_t base = C.sym.size();
        C.sym.resize(base + line.size());
        char* w = C.sym.data() + base;
        for (char c : line) {
            const uint8_t t = cls[static_cast<unsigned char>(c)];
            if (t < kSkip) {
                *w++ = char(t);
            } else if (t == kBad) {
                C.sym.resize(size_t(w - C.sym.data()));
                C.fail = {XB_PARSE_INVALID_SYMBOL, lineno,
                          "symbol '" + std::string(1, c) + "' on line " + L(lineno) +
                              " is not in the allowed alphabet"};
                return false;
            }
        }
        C.sym.resize(size_t(w - C.sym.data()));
        return true;
    });
    if (C.fail.kind == XB_PARSE_OK && have) {
        C.rec_end.push_back(int64_t(C.sym.size()));
        C.last_empty = int64_t(C.sym.size()) == rec_start;
    }
}

int64_t count_lines(std::string_view t) {
    int64_t n = 0;
    const char* p = t.data();
    const char* e = t.data() + t.size();
    while ((p = static_cast<const char*>(std::memchr(p, '\n', size_t(e - p))))) {
        ++n;
        ++p;
    }
    return n;
}

}  // namespace

struct xb_fasta {
    std::vector<char> sym;
    std::vector<int64_t> off{0};
    std::vector<char> names;
    std::vector<int64_t> name_off{0};
};

extern "C" {

xb_fasta* xb_fasta_parse(const char* text, int64_t len, const char* allowed, int n_threads,
                         xb_parse_error* err) {
    clear_err(err);
    if ((!text && len) || len < 0 || !allowed) {
        set_err(err, {XB_PARSE_BAD_ARGUMENT, 0, "invalid argument"});
        return nullptr;
    }
    uint8_t cls[256];
    fasta_classes(allowed, cls);
    const std::string_view all(text, size_t(len));
    // chunks cut just after a '\n' that precedes a '>' (each later chunk
    // starts with a header line)
    int T = n_threads > 0 ? n_threads : int(std::max(1u, std::thread::hardware_concurrency()));
    T = int(std::min<int64_t>(T, std::max<int64_t>(1, len >> 22)));  // >= 4 MB per chunk
    std::vector<size_t> cut{0};
    for (int c = 1; c < T; ++c) {
        size_t at = std::max(cut.back(), size_t(len) * size_t(c) / size_t(T));
        size_t q = all.find("\n>", at);
        if (q == std::string_view::npos) break;
        if (q + 1 > cut.back()) cut.push_back(q + 1);
    }
    cut.push_back(size_t(len));
    const size_t nc = cut.size() - 1;
    std::vector<FastaChunk> ch(nc);
    std::vector<int64_t> lines(nc, 0);
    {
        std::vector<std::thread> th;
        for (size_t c = 0; c < nc; ++c)
            th.emplace_back([&, c] { lines[c] = count_lines(all.substr(cut[c], cut[c + 1] - cut[c])); });
        for (auto& t : th) t.join();
    }
    int64_t first = 1;
    for (size_t c = 0; c < nc; ++c) {
        ch[c].text = all.substr(cut[c], cut[c + 1] - cut[c]);
        ch[c].first_line = first;
        first += lines[c];
    }
    {
        std::vector<std::thread> th;
        for (size_t c = 0; c < nc; ++c) th.emplace_back([&, c] { parse_fasta_chunk(ch[c], cls); });
        for (auto& t : th) t.join();
    }
    // errors in line order: the previous chunk's empty last record is found at
    // this chunk's first header, before anything inside this chunk
    for (size_t c = 0; c < nc; ++c) {
        if (c > 0 && ch[c - 1].fail.kind == XB_PARSE_OK && ch[c - 1].last_empty) {
            set_err(err, {XB_PARSE_EMPTY_RECORD, 0,
                          "record '" + ch[c - 1].names.back() + "' has no sequence data"});
            return nullptr;
        }
        if (ch[c].fail.kind != XB_PARSE_OK) {
            set_err(err, ch[c].fail);
            return nullptr;
        }
    }
    if (nc && ch[nc - 1].last_empty) {  // io.cpp:91-92
        set_err(err, {XB_PARSE_EMPTY_RECORD, 0, "record '" + ch[nc - 1].names.back() + "' has no sequence data"});
        return nullptr;
    }
    auto* F = new xb_fasta();
    size_t ns = 0, nr = 0, nb = 0;
    for (auto& c : ch) {
        ns += c.sym.size();
        nr += c.rec_end.size();
        for (auto& n : c.names) nb += n.size();
    }
    F->sym.resize(ns);
    F->off.reserve(nr + 1);
    F->names.reserve(nb);
    F->name_off.reserve(nr + 1);
    size_t base = 0;
    for (auto& c : ch) {
        std::memcpy(F->sym.data() + base, c.sym.data(), c.sym.size());
        for (int64_t e : c.rec_end) F->off.push_back(int64_t(base) + e);
        for (auto& n : c.names) {
            F->names.insert(F->names.end(), n.begin(), n.end());
            F->name_off.push_back(int64_t(F->names.size()));
        }
        base += c.sym.size();
    }
    return F;
}

void xb_fasta_sizes(const xb_fasta* f, int64_t* sizes3) {
    sizes3[0] = int64_t(f->off.size()) - 1;
    sizes3[1] = int64_t(f->sym.size());
    sizes3[2] = int64_t(f->names.size());
}

void xb_fasta_copy(const xb_fasta* f, char* symbols, int64_t* offsets, char* names, int64_t* name_offsets) {
    if (symbols) std::memcpy(symbols, f->sym.data(), f->sym.size());
    if (offsets) std::memcpy(offsets, f->off.data(), f->off.size() * 8);
    if (names) std::memcpy(names, f->names.data(), f->names.size());
    if (name_offsets) std::memcpy(name_offsets, f->name_off.data(), f->name_off.size() * 8);
}

int64_t xb_pool_add_fasta(xb_pool* p, const xb_fasta* f) {
    if (!p || !f) return -XB_E_BAD_PARAM;
    return xb_pool_add_bulk(p, f->sym.data(), f->off.data(), int64_t(f->off.size()) - 1);
}

void xb_fasta_free(xb_fasta* f) { delete f; }

// parse_seeds (io.cpp:98-127)
int64_t xb_parse_seeds(const char* text, int64_t len, xb_task* out, int64_t cap, xb_parse_error* err) {
    clear_err(err);
    if ((!text && len) || len < 0 || cap < 0 || (cap && !out)) {
        set_err(err, {XB_PARSE_BAD_ARGUMENT, 0, "invalid argument"});
        return -XB_E_BAD_PARAM;
    }
    int64_t n = 0;
    ParseFail fail;
    std::vector<std::string_view> toks;
    for_lines(std::string_view(text, size_t(len)), 1, [&](std::string_view line, int64_t lineno) {
        split_ws(line, toks);
        if (toks.empty() || toks[0][0] == '#') return true;
        if (toks.size() != 4) {
            fail = {XB_PARSE_MALFORMED_LINE, lineno,
                    "line " + L(lineno) + ": expected 4 fields, got " + L(int64_t(toks.size()))};
            return false;
        }
        long long f[4];
        for (int i = 0; i < 4; ++i)
            if (!parse_ll(toks[size_t(i)], f[i])) {
                fail = {XB_PARSE_MALFORMED_LINE, lineno,
                        "line " + L(lineno) + ": field '" + std::string(toks[size_t(i)]) + "' is not an integer"};
                return false;
            }
        for (int i = 0; i < 4; ++i)
            if (f[i] < 0) {
                fail = {XB_PARSE_NEGATIVE_INDEX, 0, "line " + L(lineno) + ": negative value " + L(f[i])};
                return false;
            }
        if (n < cap) out[n] = xb_task{int32_t(n), uint32_t(f[0]), uint32_t(f[1]), uint64_t(f[2]), uint64_t(f[3])};
        ++n;
        return true;
    });
    if (fail.kind != XB_PARSE_OK) {
        set_err(err, fail);
        return -XB_E_PARSE;
    }
    return n;
}

// parse_overlaps (io.cpp:129-196): Matrix Market coordinate, pattern or integer
int64_t xb_parse_overlaps(const char* text, int64_t len, xb_task* out, int64_t cap, xb_parse_error* err) {
    clear_err(err);
    if ((!text && len) || len < 0 || cap < 0 || (cap && !out)) {
        set_err(err, {XB_PARSE_BAD_ARGUMENT, 0, "invalid argument"});
        return -XB_E_BAD_PARAM;
    }
    bool saw_banner = false, saw_size = false, pattern = false;
    long long rows = 0, cols = 0, nnz = 0;
    int64_t n = 0;
    ParseFail fail;
    std::vector<std::string_view> toks;
    for_lines(std::string_view(text, size_t(len)), 1, [&](std::string_view line, int64_t lineno) {
        if (line.empty()) return true;
        if (!saw_banner) {
            split_ws(line, toks);
            if (toks.size() < 5 || toks[0] != "%%MatrixMarket" || toks[1] != "matrix" ||
                toks[2] != "coordinate" || toks[4] != "general") {
                fail = {XB_PARSE_BAD_HEADER, 0,
                        "line " + L(lineno) +
                            ": expected '%%MatrixMarket matrix coordinate {pattern|integer} general'"};
                return false;
            }
            if (toks[3] == "pattern") {
                pattern = true;
            } else if (toks[3] != "integer") {
                fail = {XB_PARSE_BAD_HEADER, 0, "unsupported field type '" + std::string(toks[3]) + "'"};
                return false;
            }
            saw_banner = true;
            return true;
        }
        if (line[0] == '%') return true;
        split_ws(line, toks);
        if (toks.empty()) return true;
        if (!saw_size) {
            long long f[3];
            if (toks.size() != 3 || !parse_ll(toks[0], f[0]) || !parse_ll(toks[1], f[1]) ||
                !parse_ll(toks[2], f[2])) {
                fail = {XB_PARSE_BAD_HEADER, 0, "line " + L(lineno) + ": expected 'rows cols entries'"};
                return false;
            }
            rows = f[0];
            cols = f[1];
            nnz = f[2];
            saw_size = true;
            return true;
        }
        const size_t want = pattern ? 2 : 4;
        if (toks.size() != want) {
            fail = {XB_PARSE_BAD_HEADER, 0,
                    "line " + L(lineno) + ": expected " + L(int64_t(want)) + " fields per entry, got " +
                        L(int64_t(toks.size())) + (pattern ? "" : " (two seed position values required)")};
            return false;
        }
        long long f[4] = {0, 0, 0, 0};
        for (size_t i = 0; i < want; ++i)
            if (!parse_ll(toks[i], f[i])) {
                fail = {XB_PARSE_BAD_HEADER, 0,
                        "line " + L(lineno) + ": field '" + std::string(toks[i]) + "' is not an integer"};
                return false;
            }
        if (f[0] < 1 || f[0] > rows || f[1] < 1 || f[1] > cols) {
            fail = {XB_PARSE_OUT_OF_SHAPE, 0,
                    "line " + L(lineno) + ": entry (" + L(f[0]) + ", " + L(f[1]) + ") outside declared " +
                        L(rows) + "x" + L(cols)};
            return false;
        }
        if (f[2] < 0 || f[3] < 0) {
            fail = {XB_PARSE_NEGATIVE_INDEX, 0, "line " + L(lineno) + ": negative seed position"};
            return false;
        }
        if (n < cap)
            out[n] = xb_task{int32_t(n), uint32_t(f[0] - 1), uint32_t(f[1] - 1), uint64_t(f[2]), uint64_t(f[3])};
        ++n;
        return true;
    });
    if (fail.kind == XB_PARSE_OK) {
        if (!saw_banner)
            fail = {XB_PARSE_BAD_HEADER, 0, "missing %%MatrixMarket banner"};
        else if (!saw_size)
            fail = {XB_PARSE_BAD_HEADER, 0, "missing size line"};
        else if ((long long)n != nnz)
            fail = {XB_PARSE_BAD_HEADER, 0, "declared " + L(nnz) + " entries, found " + L(n)};
    }
    if (fail.kind != XB_PARSE_OK) {
        set_err(err, fail);
        return -XB_E_PARSE;
    }
    return n;
}

}  // extern "C"
