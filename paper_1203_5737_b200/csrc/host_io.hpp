// Host-side CSR assembly and Matrix Market I/O for the Python module.
//
// Behaviour (accepted inputs, results, error classes and messages) follows the
// reference: csr_from_triplets (proj/src/core.cpp:7-48), read_matrix_market /
// write_matrix_market (proj/src/io.cpp:43-160).  The implementation is this
// repo's own: the whole stream is read once into memory and scanned with a
// line cursor and strtoll/strtod, the banner qualifiers are classified through
// small tables, and the CSR is assembled by a keyed sort followed by a
// count / scan / fill pass.
#pragma once

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <numeric>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "argcsr_gpu.hpp"

namespace argcsr_b200::host_io {

struct Entry {
    std::size_t row, col;
    double value;
};

// CSR from (row, col, value) entries: dimensions >= 1x1 (DimensionError),
// every entry inside (BoundsError), entries ordered by (row, col), duplicates
// accumulated left to right in that order, explicit zeros kept.
//
// The order of equal keys decides the rounding of a duplicate sum, so the
// keyed sort must make the same choices as the reference's std::sort over
// (row, col) (core.cpp:20-22): std::sort's element moves depend only on the
// comparison outcomes, and comparing packed (row, col) keys gives the same
// outcomes as comparing the pairs lexicographically, so sorting (key, value)
// records by key reproduces the reference's arrangement of equal-key values.
inline CsrMatrix assemble_csr(std::size_t num_rows, std::size_t num_cols, const std::vector<Entry>& entries) {
    if (num_rows == 0 || num_cols == 0)
        throw DimensionError("csr_from_triplets: matrix dimensions must be at least 1x1");
    struct Keyed {
        unsigned __int128 key;
        double value;
    };
    std::vector<Keyed> recs;
    recs.reserve(entries.size());
    for (const Entry& e : entries) {
        if (e.row >= num_rows || e.col >= num_cols)
            throw BoundsError("csr_from_triplets: entry (" + std::to_string(e.row) + ", " + std::to_string(e.col) +
                              ") outside " + std::to_string(num_rows) + "x" + std::to_string(num_cols));
        recs.push_back({(static_cast<unsigned __int128>(e.row) << 64) | e.col, e.value});
    }
    std::sort(recs.begin(), recs.end(), [](const Keyed& a, const Keyed& b) { return a.key < b.key; });

    // run heads: the first record of every distinct key
    std::vector<std::size_t> heads;
    heads.reserve(recs.size());
    for (std::size_t k = 0; k < recs.size(); ++k)
        if (k == 0 || recs[k].key != recs[k - 1].key) heads.push_back(k);

    CsrMatrix A;
    A.num_rows = num_rows;
    A.num_cols = num_cols;
    A.row_pointers.assign(num_rows + 1, 0);
    A.columns.resize(heads.size());
    A.values.resize(heads.size());
    for (std::size_t h = 0; h < heads.size(); ++h) {
        const std::size_t first = heads[h];
        const std::size_t last = h + 1 < heads.size() ? heads[h + 1] : recs.size();
        double acc = recs[first].value;
        for (std::size_t k = first + 1; k < last; ++k) acc += recs[k].value;
        const std::size_t row = static_cast<std::size_t>(recs[first].key >> 64);
        A.values[h] = acc;
        A.columns[h] = static_cast<index_t>(static_cast<uint64_t>(recs[first].key));
        ++A.row_pointers[row + 1];
    }
    std::partial_sum(A.row_pointers.begin(), A.row_pointers.end(), A.row_pointers.begin());
    return A;
}

// ------------------------------------------------------------ Matrix Market
namespace detail {

// A cursor over the lines of an in-memory text.
class Lines {
   public:
    explicit Lines(std::string text) : text_(std::move(text)) {}
    // next line (without the newline); false at the end
    bool next(std::string_view& out) {
        if (pos_ >= text_.size()) return false;
        const std::size_t nl = text_.find('\n', pos_);
        const std::size_t end = nl == std::string::npos ? text_.size() : nl;
        out = std::string_view(text_).substr(pos_, end - pos_);
        pos_ = end + 1;
        return true;
    }
    // next line holding data: not blank, not a '%' comment
    bool next_data(std::string_view& out) {
        while (next(out)) {
            std::size_t i = 0;
            while (i < out.size() && std::isspace(static_cast<unsigned char>(out[i]))) ++i;
            if (i < out.size() && out[i] != '%') return true;
        }
        return false;
    }
    bool empty_text() const { return text_.empty(); }

   private:
    std::string text_;
    std::size_t pos_ = 0;
};

inline std::vector<std::string> tokens(std::string_view line) {
    std::vector<std::string> t;
    std::size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        const std::size_t b = i;
        while (i < line.size() && !std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        if (i > b) t.emplace_back(line.substr(b, i - b));
    }
    return t;
}

inline std::string folded(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return char(std::tolower(c)); });
    return s;
}

// Numeric fields parsed in place like stream extraction: leading blanks
// skipped, the longest numeric prefix taken, the rest left for the next field.
class Fields {
   public:
    explicit Fields(std::string_view line) : buf_(line) {}
    bool integer(long long& v) {
        skip();
        if (pos_ >= buf_.size()) return false;
        const char* b = buf_.c_str() + pos_;
        char* e = nullptr;
        errno = 0;
        const long long r = std::strtoll(b, &e, 10);
        if (e == b || errno == ERANGE) return false;
        v = r;
        pos_ += std::size_t(e - b);
        return true;
    }
    bool real(double& v) {
        skip();
        if (pos_ >= buf_.size()) return false;
        const char* b = buf_.c_str() + pos_;
        if (!(std::isdigit(static_cast<unsigned char>(*b)) || *b == '+' || *b == '-' || *b == '.')) return false;
        char* e = nullptr;
        const double r = std::strtod(b, &e);
        if (e == b) return false;
        v = r;
        pos_ += std::size_t(e - b);
        return true;
    }

   private:
    void skip() {
        while (pos_ < buf_.size() && std::isspace(static_cast<unsigned char>(buf_[pos_]))) ++pos_;
    }
    std::string buf_;
    std::size_t pos_ = 0;
};

enum class Field { real, pattern };
enum class Symmetry { general, symmetric, skew };

struct Banner {
    Field field;
    Symmetry symmetry;
};

// The banner "%%MatrixMarket matrix coordinate <field> <symmetry>" with the
// reference's classification of every qualifier: accepted, recognised but
// unsupported (UnsupportedError), or unknown (ParseError).
inline Banner parse_banner(std::string_view line) {
    const std::vector<std::string> t = tokens(line);
    if (t.size() < 5 || folded(t[0]) != "%%matrixmarket") throw ParseError("matrix market: malformed header line");
    const std::string object = folded(t[1]), format = folded(t[2]), field = folded(t[3]), sym = folded(t[4]);
    if (object != "matrix") throw UnsupportedError("matrix market: object '" + object + "' not supported");
    if (format == "array") throw UnsupportedError("matrix market: array format not supported");
    if (format != "coordinate") throw ParseError("matrix market: unknown format '" + format + "'");

    static const std::pair<const char*, Field> kFields[] = {
        {"real", Field::real}, {"integer", Field::real}, {"pattern", Field::pattern}};
    static const std::pair<const char*, Symmetry> kSym[] = {
        {"general", Symmetry::general}, {"symmetric", Symmetry::symmetric}, {"skew-symmetric", Symmetry::skew}};
    Banner b{};
    bool have_field = false, have_sym = false;
    for (const auto& [name, f] : kFields)
        if (field == name) b.field = f, have_field = true;
    if (!have_field) {
        if (field == "complex") throw UnsupportedError("matrix market: complex field not supported");
        throw ParseError("matrix market: unknown field '" + field + "'");
    }
    for (const auto& [name, s] : kSym)
        if (sym == name) b.symmetry = s, have_sym = true;
    if (!have_sym) {
        if (sym == "hermitian") throw UnsupportedError("matrix market: hermitian symmetry not supported");
        throw ParseError("matrix market: unknown symmetry '" + sym + "'");
    }
    return b;
}

}  // namespace detail

inline CsrMatrix parse_matrix_market(std::string text) {
    using namespace detail;
    Lines lines(std::move(text));
    std::string_view line;
    if (lines.empty_text() || !lines.next(line)) throw ParseError("matrix market: empty stream");
    const Banner banner = parse_banner(line);

    if (!lines.next_data(line)) throw ParseError("matrix market: missing size line");
    long long dims[3] = {0, 0, 0};
    {
        Fields f(line);
        for (long long& d : dims)
            if (!f.integer(d) || d < 0) throw ParseError("matrix market: malformed size line '" + std::string(line) + "'");
    }
    const long long rows = dims[0], cols = dims[1], count = dims[2];
    if (rows == 0 || cols == 0) throw ParseError("matrix market: matrix dimensions must be positive");

    const bool mirrored = banner.symmetry != Symmetry::general;
    std::vector<Entry> entries;
    entries.reserve(std::size_t(count) * (mirrored ? 2 : 1));
    for (long long k = 0; k < count; ++k) {
        if (!lines.next_data(line))
            throw ParseError("matrix market: expected " + std::to_string(count) + " entries, got " + std::to_string(k));
        Fields f(line);
        long long i = 0, j = 0;
        double v = 1.0;  // pattern entries are ones
        if (!f.integer(i) || !f.integer(j)) throw ParseError("matrix market: malformed entry '" + std::string(line) + "'");
        if (banner.field == Field::real && !f.real(v))
            throw ParseError("matrix market: entry missing value '" + std::string(line) + "'");
        if (i < 1 || j < 1 || i > rows || j > cols)
            throw BoundsError("matrix market: entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside " +
                              std::to_string(rows) + "x" + std::to_string(cols));
        entries.push_back({std::size_t(i - 1), std::size_t(j - 1), v});
        if (mirrored && i != j)
            entries.push_back({std::size_t(j - 1), std::size_t(i - 1), banner.symmetry == Symmetry::skew ? -v : v});
    }
    return assemble_csr(std::size_t(rows), std::size_t(cols), entries);
}

inline CsrMatrix read_matrix_market_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_matrix_market(std::move(text));
}

// "%%MatrixMarket matrix coordinate real general", the size line, then one
// 1-based "row col value" line per stored entry in row order, values with 17
// significant digits (round-trips every double).
inline void write_matrix_market_file(const std::string& path, const CsrMatrix& A) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw IoError("cannot open '" + path + "' for writing");
    bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%zu %zu %zu\n", A.num_rows,
                           A.num_cols, A.nnz()) > 0;
    for (std::size_t r = 0; ok && r < A.num_rows; ++r)
        for (std::size_t k = A.row_pointers[r]; ok && k < A.row_pointers[r + 1]; ++k)
            ok = std::fprintf(f, "%zu %lld %.17g\n", r + 1, static_cast<long long>(A.columns[k]) + 1, A.values[k]) > 0;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw IoError("matrix market: write failure");
}

}  // namespace argcsr_b200::host_io
