// Matrix Market ingestion ("a Matrix Market reader feeding
// device CSR").  Mirrors amgreuse::mm_read / mm_read_vector
// (proj/src/matrix_market.cpp:104-203, same accepted formats and error texts)
// and assembles the CSR on the device exactly like csr_from_triplets
// (proj/src/csr.cpp:24-75): entries stably bucketed by row in input order,
// stably sorted by column, duplicates summed left to right starting from the
// first value.  The text is parsed on the host by several threads (chunks
// split at line boundaries); the triplets go to the device once, where a
// stable radix sort on (row, column) keys and a per-key sequential sum build
// the matrix.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "hierarchy.cuh"

struct amgr_matrix {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    amgr::DevArray<int> rp, col;
    amgr::DevArray<double> val;
};

namespace amgr {
namespace {

[[noreturn]] void parse_fail(const std::string& path, int64_t line, const std::string& msg) {
    std::ostringstream os;
    os << path << ":" << line << ": " << msg;
    fail(AMGR_E_RUNTIME, os.str());
}

std::string lower(std::string s) {
    std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    return s;
}

struct Text {
    std::string path, buf;
    // line cursor
    size_t pos = 0;
    int64_t line_no = 0;
    bool next_line(std::string_view& out) {  // any line (banner)
        if (pos >= buf.size()) return false;
        size_t e = buf.find('\n', pos);
        if (e == std::string::npos) e = buf.size();
        out = std::string_view(buf).substr(pos, e - pos);
        pos = e + 1;
        ++line_no;
        return true;
    }
    // next non-comment, non-blank line (matrix_market.cpp:77-88)
    bool next_data_line(std::string_view& out) {
        std::string_view l;
        while (next_line(l)) {
            const size_t f = l.find_first_not_of(" \t\r");
            if (f == std::string_view::npos) continue;
            if (l[f] == '%') continue;
            out = l;
            return true;
        }
        return false;
    }
};

Text load(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(AMGR_E_RUNTIME, "cannot open file: " + path);
    Text t;
    t.path = path;
    std::ostringstream ss;
    ss << in.rdbuf();
    t.buf = ss.str();
    return t;
}

struct Header {
    std::string object, format, field, symmetry;
};

// banner checks (matrix_market.cpp:40-63)
Header banner(Text& t) {
    std::string_view l;
    if (!t.next_line(l)) parse_fail(t.path, 1, "empty file");
    std::istringstream hs{std::string(l)};
    std::string tag;
    Header h;
    hs >> tag >> h.object >> h.format >> h.field >> h.symmetry;
    if (lower(tag) != "%%matrixmarket") parse_fail(t.path, 1, "missing MatrixMarket banner");
    h.object = lower(h.object);
    h.format = lower(h.format);
    h.field = lower(h.field);
    h.symmetry = lower(h.symmetry);
    if (h.object != "matrix") parse_fail(t.path, 1, "unsupported object: " + h.object);
    if (h.field == "complex" || h.field == "pattern")
        parse_fail(t.path, 1, "unsupported format: field '" + h.field + "'");
    if (h.field != "real" && h.field != "integer") parse_fail(t.path, 1, "unsupported field: " + h.field);
    if (h.symmetry != "general" && h.symmetry != "symmetric")
        parse_fail(t.path, 1, "unsupported symmetry: " + h.symmetry);
    return h;
}

// whitespace tokens of a line (istream >> semantics for the fields we read)
int tokens(std::string_view l, std::string_view* out, int maxn) {
    int k = 0;
    size_t p = 0;
    while (k < maxn) {
        p = l.find_first_not_of(" \t\r\v\f", p);
        if (p == std::string_view::npos) break;
        size_t e = l.find_first_of(" \t\r\v\f", p);
        if (e == std::string_view::npos) e = l.size();
        out[k++] = l.substr(p, e - p);
        p = e;
    }
    return k;
}

// istream extraction semantics for `ss >> i >> j >> vtok`
// (matrix_market.cpp:124): integers are the longest [+-]digits prefix after
// whitespace and the stream continues right after it ("2 2.5 1" reads
// i = 2, j = 2, vtok = ".5"); the token is the next whitespace-free run.
struct Cursor {
    std::string_view s;
    size_t p = 0;
    void ws() {
        while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
    }
    bool read_int(int64_t& v) {
        ws();
        size_t q = p;
        if (q < s.size() && (s[q] == '+' || s[q] == '-')) ++q;
        const size_t d = q;
        while (q < s.size() && std::isdigit(static_cast<unsigned char>(s[q]))) ++q;
        if (q == d) return false;
        std::string tmp(s.substr(p, q - p));
        errno = 0;
        const long long x = std::strtoll(tmp.c_str(), nullptr, 10);
        if (errno == ERANGE) return false;
        v = x;
        p = q;
        return true;
    }
    bool read_token(std::string_view& t) {
        ws();
        if (p >= s.size()) return false;
        size_t q = p;
        while (q < s.size() && !std::isspace(static_cast<unsigned char>(s[q]))) ++q;
        t = s.substr(p, q - p);
        p = q;
        return true;
    }
};

// std::stod with the reference's full-token check (matrix_market.cpp:95-106);
// stod throws (-> "non-numeric value") on no conversion and on ERANGE
bool parse_double(std::string_view s, double& v) {
    std::string tmp(s);
    char* end = nullptr;
    errno = 0;
    v = std::strtod(tmp.c_str(), &end);
    return end != tmp.c_str() && *end == '\0' && errno != ERANGE;
}

struct Chunk {
    std::vector<int> row, col;
    std::vector<double> val;
    std::string err;
    int64_t err_line = 0;
};

__global__ void k_mm_keys(int64_t m, const int* __restrict__ row, const int* __restrict__ col, int bc,
                          uint64_t* key, int* id) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < m;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        key[t] = (static_cast<uint64_t>(row[t]) << bc) | static_cast<uint64_t>(col[t]);
        id[t] = static_cast<int>(t);
    }
}

__global__ void k_mm_heads(int64_t m, const uint64_t* __restrict__ k, int64_t* head) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < m;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        head[t] = (t == 0 || k[t] != k[t - 1]) ? 1 : 0;
}

// unique key u: first sorted position s0; value = v0 + v1 + ... in input order
__global__ void k_mm_assemble(int64_t m, const uint64_t* __restrict__ k, const int* __restrict__ perm,
                              const int64_t* __restrict__ head, const int64_t* __restrict__ pos,
                              const double* __restrict__ v, uint64_t mask, int* col, double* val,
                              uint64_t* ukeys) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < m;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!head[t]) continue;
        const int64_t u = pos[t];
        double s = v[perm[t]];
        for (int64_t q = t + 1; q < m && !head[q]; ++q) s = __dadd_rn(s, v[perm[q]]);
        val[u] = s;
        col[u] = static_cast<int>(k[t] & mask);
        ukeys[u] = k[t];
    }
}

__global__ void k_mm_rowptr(const uint64_t* ukeys, int64_t nnz, int64_t n, int bc, int* rp) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t target = static_cast<uint64_t>(i) << bc;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        rp[i] = static_cast<int>(lo);
    }
}

int bits(int64_t n) {
    int b = 1;
    while ((int64_t{1} << b) < n) ++b;
    return b;
}

}  // namespace

// Device assembly exactly as csr_from_triplets (csr.cpp:24-75): stable
// radix sort of (row, col) keys (duplicates keep input order) and an in-order
// segmented sum of duplicates.
void assemble_triplets(Ctx& c, int64_t nrows, int64_t ncols, const std::vector<int>& row, const std::vector<int>& col,
                       const std::vector<double>& val, amgr_matrix& M) {
    const int64_t m = static_cast<int64_t>(row.size());
    M.nrows = nrows;
    M.ncols = ncols;
    M.rp.alloc(nrows + 1, c.stream);
    const int bc = bits(std::max<int64_t>(ncols, 2)), br = bits(std::max<int64_t>(nrows, 2));
    if (m == 0) {
        CK(cudaMemsetAsync(M.rp.get(), 0, sizeof(int) * (nrows + 1), c.stream));
        M.nnz = 0;
        M.col.alloc(1, c.stream);
        M.val.alloc(1, c.stream);
        CK(cudaStreamSynchronize(c.stream));
        return;
    }
    DevArray<int> drow(m, c.stream), dcol(m, c.stream), id0(m, c.stream), id1(m, c.stream);
    DevArray<double> dval(m, c.stream);
    DevArray<uint64_t> k0(m, c.stream), k1(m, c.stream);
    h2d(drow.get(), row.data(), m, c.stream);
    h2d(dcol.get(), col.data(), m, c.stream);
    h2d(dval.get(), val.data(), m, c.stream);
    LAUNCH(c, "io", 0.0, k_mm_keys, grid_for(m, 256, c.num_sms * 16), 256, 0, m, drow.get(), dcol.get(), bc, k0.get(),
           id0.get());
    cub::DoubleBuffer<uint64_t> kb(k0.get(), k1.get());
    cub::DoubleBuffer<int> vb(id0.get(), id1.get());
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, m, 0, br + bc, c.stream));
    {
        DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
        CK(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kb, vb, m, 0, br + bc, c.stream));
    }
    DevArray<int64_t> head(m, c.stream), pos(m, c.stream);
    LAUNCH(c, "io", 0.0, k_mm_heads, grid_for(m, 256, c.num_sms * 16), 256, 0, m, kb.Current(), head.get());
    bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, head.get(), pos.get(), m, c.stream));
    {
        DevArray<char> tmp(static_cast<int64_t>(bytes), c.stream);
        CK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, head.get(), pos.get(), m, c.stream));
    }
    const int64_t nu = d2h_scalar(pos.get() + m - 1, c.stream) + d2h_scalar(head.get() + m - 1, c.stream);
    M.nnz = nu;
    M.col.alloc(nu, c.stream);
    M.val.alloc(nu, c.stream);
    DevArray<uint64_t> uk(nu, c.stream);
    LAUNCH(c, "io", 0.0, k_mm_assemble, grid_for(m, 256, c.num_sms * 16), 256, 0, m, kb.Current(), vb.Current(),
           head.get(), pos.get(), dval.get(), (uint64_t{1} << bc) - 1, M.col.get(), M.val.get(), uk.get());
    LAUNCH(c, "io", 0.0, k_mm_rowptr, grid_for(nrows + 1, 256, c.num_sms * 16), 256, 0, uk.get(), nu, nrows, bc,
           M.rp.get());
    CK(cudaStreamSynchronize(c.stream));
}

// mm_read (matrix_market.cpp:104-140) into device CSR
void mm_read_device(Ctx& c, const std::string& path, amgr_matrix& M) {
    Text t = load(path);
    const Header h = banner(t);
    if (h.format != "coordinate") parse_fail(path, 1, "expected coordinate format, got " + h.format);
    const bool symmetric = h.symmetry == "symmetric";
    std::string_view line;
    if (!t.next_data_line(line)) parse_fail(path, t.line_no, "missing size line");
    int64_t nrows = 0, ncols = 0, nnz = 0;
    {
        std::istringstream ss{std::string(line)};
        if (!(ss >> nrows >> ncols >> nnz) || nrows < 0 || ncols < 0 || nnz < 0)
            parse_fail(path, t.line_no, "malformed size line '" + std::string(line) + "'");
    }
    if (nrows >= (int64_t{1} << 31) || ncols >= (int64_t{1} << 31) || (symmetric ? 2 : 1) * nnz >= (int64_t{1} << 31))
        fail(AMGR_E_RUNTIME, "mm_read: matrix exceeds the int32 index range of the device CSR");
    // split the rest of the file into chunks at line boundaries; parse in
    // parallel; the first error in file order wins (line numbers from counts)
    const size_t body = t.pos, total = t.buf.size();
    const int nthreads = static_cast<int>(std::max<size_t>(1, std::min<size_t>(
        std::thread::hardware_concurrency() ? std::thread::hardware_concurrency() : 1, (total - body) / (1 << 20) + 1)));
    std::vector<size_t> cut(static_cast<size_t>(nthreads) + 1);
    cut[0] = body;
    cut[nthreads] = total;
    for (int k = 1; k < nthreads; ++k) {
        size_t p = body + (total - body) * k / nthreads;
        while (p < total && t.buf[p - 1] != '\n') ++p;
        cut[k] = std::max(p, cut[k - 1]);
    }
    std::vector<Chunk> ch(static_cast<size_t>(nthreads));
    std::vector<int64_t> lines_in(static_cast<size_t>(nthreads), 0), entries_in(static_cast<size_t>(nthreads), 0);
    auto work = [&](int k) {
        Chunk& C = ch[k];
        std::string_view s = std::string_view(t.buf).substr(cut[k], cut[k + 1] - cut[k]);
        size_t p = 0;
        int64_t ln = 0;
        while (p < s.size()) {
            size_t e = s.find('\n', p);
            if (e == std::string_view::npos) e = s.size();
            std::string_view l = s.substr(p, e - p);
            p = e + 1;
            ++ln;
            const size_t f = l.find_first_not_of(" \t\r");
            if (f == std::string_view::npos || l[f] == '%') continue;
            Cursor cur{l};
            std::string_view vtok;
            int64_t i = 0, j = 0;
            double v = 0.0;
            auto bad = [&](const std::string& msg) {
                C.err = msg;
                C.err_line = ln;
            };
            if (!cur.read_int(i) || !cur.read_int(j) || !cur.read_token(vtok)) {
                bad("malformed entry '" + std::string(l) + "'");
                break;
            }
            if (i < 1 || i > nrows || j < 1 || j > ncols) {
                std::ostringstream os;
                os << "index (" << i << ", " << j << ") out of declared bounds " << nrows << "x" << ncols;
                bad(os.str());
                break;
            }
            if (!parse_double(vtok, v)) {
                bad("non-numeric value '" + std::string(vtok) + "'");
                break;
            }
            C.row.push_back(static_cast<int>(i - 1));
            C.col.push_back(static_cast<int>(j - 1));
            C.val.push_back(v);
            if (symmetric && i != j) {
                C.row.push_back(static_cast<int>(j - 1));
                C.col.push_back(static_cast<int>(i - 1));
                C.val.push_back(v);
            }
            ++entries_in[k];
        }
        lines_in[k] = ln;
    };
    {
        std::vector<std::thread> th;
        for (int k = 1; k < nthreads; ++k) th.emplace_back(work, k);
        work(0);
        for (auto& x : th) x.join();
    }
    // walk the chunks in file order: entries beyond nnz are ignored, an error
    // counts only if it occurs before the nnz-th entry (the reference stops
    // reading after nnz entries)
    std::vector<int> row, col;
    std::vector<double> val;
    row.reserve(static_cast<size_t>(symmetric ? 2 * nnz : nnz));
    col.reserve(row.capacity());
    val.reserve(row.capacity());
    int64_t taken = 0, line_base = t.line_no;
    for (int k = 0; k < nthreads && taken < nnz; ++k) {
        Chunk& C = ch[k];
        // replay this chunk's entries up to nnz
        size_t q = 0;
        while (q < C.row.size() && taken < nnz) {
            // entries were appended as (i,j) [+ (j,i) when symmetric and i != j]
            row.push_back(C.row[q]);
            col.push_back(C.col[q]);
            val.push_back(C.val[q]);
            if (symmetric && C.row[q] != C.col[q]) {
                row.push_back(C.row[q + 1]);
                col.push_back(C.col[q + 1]);
                val.push_back(C.val[q + 1]);
                q += 2;
            } else {
                q += 1;
            }
            ++taken;
        }
        if (taken < nnz && !C.err.empty()) parse_fail(path, line_base + C.err_line, C.err);
        line_base += lines_in[k];
    }
    if (taken < nnz) parse_fail(path, line_base, "unexpected end of file: expected more entries");

    assemble_triplets(c, nrows, ncols, row, col, val, M);
}

// mm_read_vector (matrix_market.cpp:176-203)
std::vector<double> mm_read_vector_host(const std::string& path) {
    Text t = load(path);
    const Header h = banner(t);
    if (h.format != "array") parse_fail(path, 1, "expected array format, got " + h.format);
    if (h.symmetry != "general") parse_fail(path, 1, "vectors must be general");
    std::string_view line;
    if (!t.next_data_line(line)) parse_fail(path, t.line_no, "missing size line");
    int64_t nrows = 0, ncols = 0;
    {
        std::istringstream ss{std::string(line)};
        if (!(ss >> nrows >> ncols) || nrows < 0) parse_fail(path, t.line_no, "malformed size line '" + std::string(line) + "'");
    }
    if (ncols != 1) parse_fail(path, t.line_no, "expected a single-column array");
    std::vector<double> v;
    v.reserve(static_cast<size_t>(nrows));
    for (int64_t k = 0; k < nrows; ++k) {
        if (!t.next_data_line(line)) parse_fail(path, t.line_no, "unexpected end of file: expected more entries");
        std::string_view tok[1];
        if (tokens(line, tok, 1) < 1) parse_fail(path, t.line_no, "malformed entry '" + std::string(line) + "'");
        double x = 0.0;
        if (!parse_double(tok[0], x)) parse_fail(path, t.line_no, "non-numeric value '" + std::string(tok[0]) + "'");
        v.push_back(x);
    }
    return v;
}

}  // namespace amgr

extern "C" {

amgr_status amgr_mm_read(amgr_ctx* ctx, const char* path, amgr_matrix** out) {
    if (!ctx || !path || !out) return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    amgr::Ctx& c = ctx->c;
    auto* m = new amgr_matrix();
    try {
        CK(cudaSetDevice(c.device));
        amgr::mm_read_device(c, path, *m);
        *out = m;
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        delete m;
        c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        delete m;
        c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

amgr_status amgr_csr_from_triplets(amgr_ctx* ctx, int64_t nrows, int64_t ncols, int64_t count, const int64_t* rows,
                                   const int64_t* cols, const double* values, amgr_matrix** out) {
    if (!ctx || !out || count < 0 || (count > 0 && (!rows || !cols || !values))) return AMGR_E_INVALID_ARGUMENT;
    *out = nullptr;
    amgr::Ctx& c = ctx->c;
    auto* m = new amgr_matrix();
    try {
        CK(cudaSetDevice(c.device));
        // validation in the reference's order and words (csr.cpp:25-35)
        if (nrows < 0 || ncols < 0) amgr::invalid("csr_from_triplets: negative dimension");
        if (nrows > INT32_MAX - 1 || ncols > INT32_MAX - 1 || count > INT32_MAX - 1)
            amgr::invalid("matrix too large for int32 device indices (> 2^31 entries per GPU)");
        std::vector<int> r(static_cast<size_t>(count)), cc(static_cast<size_t>(count));
        std::vector<double> v(values, values + count);
        for (int64_t k = 0; k < count; ++k) {
            if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols) {
                std::ostringstream os;
                os << "csr_from_triplets: entry " << k << " (" << rows[k] << ", " << cols[k] << ") out of range for "
                   << nrows << "x" << ncols << " matrix";
                amgr::invalid(os.str());
            }
            r[static_cast<size_t>(k)] = static_cast<int>(rows[k]);
            cc[static_cast<size_t>(k)] = static_cast<int>(cols[k]);
        }
        amgr::assemble_triplets(c, nrows, ncols, r, cc, v, *m);
        *out = m;
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        delete m;
        c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        delete m;
        c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

amgr_status amgr_matrix_csr(const amgr_matrix* m, amgr_csr* view) {
    if (!m || !view) return AMGR_E_INVALID_ARGUMENT;
    view->nrows = m->nrows;
    view->ncols = m->ncols;
    view->nnz = m->nnz;
    view->row_ptr = m->rp.get();
    view->col_idx = m->col.get();
    view->values = m->val.get();
    view->index_bits = 32;
    view->location = AMGR_DEVICE;
    return AMGR_OK;
}

void amgr_matrix_free(amgr_matrix* m) { delete m; }

amgr_status amgr_mm_read_vector(amgr_ctx* ctx, const char* path, int64_t* n, double* values) {
    if (!ctx || !path || !n) return AMGR_E_INVALID_ARGUMENT;
    amgr::Ctx& c = ctx->c;
    try {
        std::vector<double> v = amgr::mm_read_vector_host(path);
        if (values && *n >= static_cast<int64_t>(v.size())) std::copy(v.begin(), v.end(), values);
        *n = static_cast<int64_t>(v.size());
        return AMGR_OK;
    } catch (const amgr::Error& e) {
        c.last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        c.last_error = e.what();
        return AMGR_E_RUNTIME;
    }
}

}  // extern "C"
