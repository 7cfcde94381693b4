// instance_io.cu -- native parser / serializer of the instance text format
// (SURVEY.md 8(f) row 2), feeding CSR straight to the engine.
//
// Format and error behaviour follow the reference (instance.py:114-174):
//   p mhs <n> <m> [k]
//   e <demand> <v1> <v2> ...        (exactly m lines, 1-based vertices)
// '#' lines and blank lines are skipped; errors carry the 1-based line number
// ("line N: ...") and the reference's message texts.  One pass over the text,
// O(text) work, no per-edge allocations (members are appended to one CSR
// array and sorted in place per edge).  Limits: n, m < 2^31 (CSR int32).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/mhsk.h"

extern void mhsk_internal_set_error(const std::string& msg);

struct mhsk_instance {
    int32_t n = 0, m = 0;
    bool has_budget = false;
    int64_t budget = 0;
    std::vector<int64_t> ptr;
    std::vector<int32_t> vtx;
    std::vector<int32_t> dem;
};

namespace {

// Python str.split() / str.strip() whitespace (ASCII subset).
inline bool is_space(char ch) {
    return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f' ||
           (ch >= '\x1c' && ch <= '\x1f');
}
// Python str.splitlines() separators (ASCII subset).
inline bool is_newline(char ch) {
    return ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f' || (ch >= '\x1c' && ch <= '\x1e');
}

// Python int(token) for plain ASCII decimal literals: optional sign, digits,
// single underscores between digits.  Sets *big when |value| >= 2^62.
bool parse_int(const char* s, size_t len, int64_t* out, bool* big) {
    size_t i = 0;
    bool neg = false;
    *big = false;
    if (i < len && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
    if (i >= len) return false;
    int64_t v = 0;
    bool prev_digit = false;
    for (; i < len; ++i) {
        const char ch = s[i];
        if (ch >= '0' && ch <= '9') {
            if (v > ((int64_t)1 << 62) / 10) *big = true;
            else v = v * 10 + (ch - '0');
            prev_digit = true;
        } else if (ch == '_' && prev_digit && i + 1 < len && s[i + 1] >= '0' && s[i + 1] <= '9') {
            prev_digit = false;
        } else {
            return false;
        }
    }
    *out = neg ? -v : v;
    return true;
}

// Python's str(int(token)) for a literal accepted by parse_int.
std::string py_int_str(const char* s, size_t len) {
    std::string digits;
    bool neg = false;
    size_t i = 0;
    if (i < len && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
    for (; i < len; ++i)
        if (s[i] != '_') digits += s[i];
    const size_t nz = digits.find_first_not_of('0');
    digits = nz == std::string::npos ? "0" : digits.substr(nz);
    return (neg && digits != "0" ? "-" : "") + digits;
}

std::string py_repr(const std::string& t) {
    const bool sq = t.find('\'') != std::string::npos, dq = t.find('"') != std::string::npos;
    const char q = (sq && !dq) ? '"' : '\'';
    std::string r(1, q);
    for (char ch : t) {
        if (ch == '\\') r += "\\\\";
        else if (ch == q) { r += '\\'; r += ch; }
        else if (ch == '\t') r += "\\t";
        else if ((unsigned char)ch < 0x20 || ch == 0x7f) {
            char buf[8];
            snprintf(buf, sizeof buf, "\\x%02x", (unsigned char)ch);
            r += buf;
        } else r += ch;
    }
    return r + q;
}

struct Tok {
    const char* p;
    size_t len;
};

int fail(const std::string& msg, int64_t line) {
    mhsk_internal_set_error(line > 0 ? "line " + std::to_string(line) + ": " + msg : msg);
    return MHSK_INVALID;
}

}  // namespace

extern "C" {

int mhsk_parse_instance(const char* text, int64_t len, mhsk_instance** out) {
    if (!out || (!text && len > 0) || len < 0) {
        mhsk_internal_set_error("invalid arguments");
        return MHSK_INVALID;
    }
    *out = nullptr;
    mhsk_instance* inst = new mhsk_instance();
    bool have_header = false;
    int64_t header_line = 0, n = 0, m = 0;
    std::vector<Tok> toks;
    int64_t line_no = 0;
    int64_t pos = 0;
    inst->ptr.push_back(0);
    while (pos < len) {
        // one line [pos, end)
        int64_t end = pos;
        while (end < len && !is_newline(text[end])) ++end;
        ++line_no;
        const int64_t next = (end < len && text[end] == '\r' && end + 1 < len && text[end + 1] == '\n')
                                 ? end + 2
                                 : end + 1;
        // tokenize (split() on whitespace)
        toks.clear();
        for (int64_t i = pos; i < end;) {
            while (i < end && is_space(text[i])) ++i;
            if (i >= end) break;
            const int64_t s = i;
            while (i < end && !is_space(text[i])) ++i;
            toks.push_back(Tok{text + s, (size_t)(i - s)});
        }
        pos = next;
        if (toks.empty() || toks[0].p[0] == '#') continue;
        auto tok = [&](size_t k) { return std::string(toks[k].p, toks[k].len); };
        if (!have_header) {
            if (tok(0) != "p" || toks.size() < 4 || toks.size() > 5 || tok(1) != "mhs") {
                delete inst;
                return fail("expected header 'p mhs <n> <m> [k]'", line_no);
            }
            int64_t vals[3] = {0, 0, 0};
            bool big = false, any_big = false;
            for (size_t k = 2; k < toks.size(); ++k) {
                if (!parse_int(toks[k].p, toks[k].len, &vals[k - 2], &big)) {
                    delete inst;
                    return fail("non-integer field in header", line_no);
                }
                any_big |= big;
            }
            if (vals[0] < 0 || vals[1] < 0) {
                delete inst;
                return fail("vertex/edge counts must be non-negative", line_no);
            }
            if (toks.size() == 5 && vals[2] < 0) {
                delete inst;
                return fail("budget must be non-negative", line_no);
            }
            if (any_big || vals[0] > INT32_MAX || vals[1] > INT32_MAX) {
                delete inst;
                return fail("instance too large for the native engine (n, m < 2^31)", line_no);
            }
            n = vals[0];
            m = vals[1];
            inst->has_budget = toks.size() == 5;
            inst->budget = vals[2];
            have_header = true;
            header_line = line_no;
            const size_t hint = (size_t)std::min<int64_t>(m, len / 2) + 1;  // m lines need >= 2m bytes
            inst->ptr.reserve(hint);
            inst->dem.reserve(hint);
            inst->vtx.reserve((size_t)(len / 2) + 1);
            continue;
        }
        if (tok(0) != "e") {
            delete inst;
            return fail("expected edge line 'e <demand> <v1> ...', got " + py_repr(tok(0)), line_no);
        }
        if (toks.size() < 2) {
            delete inst;
            return fail("edge line missing demand", line_no);
        }
        // all fields must be integers before any other check (reference order)
        std::vector<int64_t> vals(toks.size() - 1);
        std::vector<char> huge(toks.size() - 1, 0);
        for (size_t k = 1; k < toks.size(); ++k) {
            bool big = false;
            if (!parse_int(toks[k].p, toks[k].len, &vals[k - 1], &big)) {
                delete inst;
                return fail("non-integer field in edge line", line_no);
            }
            huge[k - 1] = big;
        }
        if (huge[0] ? toks[1].p[0] == '-' : vals[0] < 1) {
            delete inst;
            return fail("demand must be positive, got " + py_int_str(toks[1].p, toks[1].len), line_no);
        }
        if (huge[0] || vals[0] > INT32_MAX) {
            delete inst;
            return fail("demand too large for the native engine", line_no);
        }
        const int64_t f = vals[0];
        const size_t base = inst->vtx.size();
        bool clean = true;
        for (size_t k = 1; k < vals.size(); ++k) {
            if (huge[k] || vals[k] < 1 || vals[k] > n) { clean = false; break; }
            inst->vtx.push_back((int32_t)(vals[k] - 1));
        }
        if (clean) {
            std::sort(inst->vtx.begin() + base, inst->vtx.end());
            clean = std::adjacent_find(inst->vtx.begin() + base, inst->vtx.end()) == inst->vtx.end();
        }
        if (!clean) {
            // report the first error in input order, as the reference does
            std::unordered_set<int64_t> seen;
            for (size_t k = 1; k < vals.size(); ++k) {
                const std::string vs = py_int_str(toks[k + 1].p, toks[k + 1].len);
                if (huge[k] || vals[k] < 1 || vals[k] > n) {
                    delete inst;
                    return fail("vertex " + vs + " out of range 1.." + std::to_string(n), line_no);
                }
                if (!seen.insert(vals[k]).second) {
                    delete inst;
                    return fail("duplicate vertex " + vs + " in edge", line_no);
                }
            }
        }
        inst->ptr.push_back((int64_t)inst->vtx.size());
        inst->dem.push_back((int32_t)f);
    }
    if (!have_header) {
        delete inst;
        return fail("missing header line", 0);
    }
    const int64_t found = (int64_t)inst->dem.size();
    if (found != m) {
        delete inst;
        return fail("header declares " + std::to_string(m) + " edges but " + std::to_string(found) +
                        " found",
                    header_line);
    }
    inst->n = (int32_t)n;
    inst->m = (int32_t)m;
    *out = inst;
    return MHSK_OK;
}

int mhsk_instance_dims(const mhsk_instance* inst, int32_t* n, int32_t* m, int64_t* nnz,
                       int32_t* has_budget, int64_t* budget) {
    if (!inst) return MHSK_INVALID;
    if (n) *n = inst->n;
    if (m) *m = inst->m;
    if (nnz) *nnz = (int64_t)inst->vtx.size();
    if (has_budget) *has_budget = inst->has_budget;
    if (budget) *budget = inst->budget;
    return MHSK_OK;
}

int mhsk_instance_copy(const mhsk_instance* inst, int64_t* edge_ptr, int32_t* edge_vtx,
                       int32_t* demand) {
    if (!inst) return MHSK_INVALID;
    if (edge_ptr) std::copy(inst->ptr.begin(), inst->ptr.end(), edge_ptr);
    if (edge_vtx) std::copy(inst->vtx.begin(), inst->vtx.end(), edge_vtx);
    if (demand) std::copy(inst->dem.begin(), inst->dem.end(), demand);
    return MHSK_OK;
}

void mhsk_instance_free(mhsk_instance* inst) { delete inst; }

int64_t mhsk_serialize_instance(int32_t n, int32_t m, const int64_t* edge_ptr,
                                const int32_t* edge_vtx, const int32_t* demand,
                                int32_t has_budget, int64_t budget, char* out, int64_t capacity) {
    // instance.py:168-174: "p mhs n m[ k]" then "e f v1 v2 ..." lines, trailing newline
    std::string s;
    s.reserve(64);
    char buf[64];
    int64_t total = 0;
    auto emit = [&](const char* p, size_t k) {
        if (out && total + (int64_t)k <= capacity) memcpy(out + total, p, k);
        total += (int64_t)k;
    };
    int k = has_budget ? snprintf(buf, sizeof buf, "p mhs %d %d %lld\n", n, m, (long long)budget)
                       : snprintf(buf, sizeof buf, "p mhs %d %d\n", n, m);
    emit(buf, (size_t)k);
    for (int32_t e = 0; e < m; ++e) {
        k = snprintf(buf, sizeof buf, "e %d", demand[e]);
        emit(buf, (size_t)k);
        for (int64_t q = edge_ptr[e]; q < edge_ptr[e + 1]; ++q) {
            k = snprintf(buf, sizeof buf, " %d", edge_vtx[q] + 1);
            emit(buf, (size_t)k);
        }
        emit("\n", 1);
    }
    return total;
}

}  // extern "C"
