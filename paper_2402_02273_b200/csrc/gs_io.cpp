// gs_io.cpp -- snapshot / metrics files and image loaders behind the C-ABI.
//
// Formats follow the reference byte for byte (paths relative to /root/reference/proj):
//   write_vtk          src/vtk.cpp:59-91     legacy ASCII VTK, one %.17g value per line
//   read_vtk           src/vtk.cpp:93-143    token reader with the reference's messages
//   write_metrics_csv  src/vtk.cpp:145-157
//   load_stack         src/imaging.cpp:14-61, 76-93   binary PGM (P5, maxval 255) slices
//   load_raw_volume    src/imaging.cpp:95-116         "nx ny nz\n" + bytes
//   write/read_label_volume  src/imaging.cpp:166-190
//
// What is B200-side about host file code: a C4 snapshot is 16.7 M values.  The reference
// formats them one snprintf at a time (~0.4 us each, ~7 s per snapshot); here an exact
// %.17g formatter (128-bit powers of ten, snprintf only on the rare near-tie) runs on a
// pool of threads feeding an ordered writer, and the GPU keeps stepping meanwhile
// (gs_snapshot_vtk in gs_capi.cu).  read_vtk parses the value region in parallel chunks.
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <climits>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <vector>

#include "gliosim_b200.h"
#include "gs_io.hpp"

namespace gsio {
void set_free_error(const std::string& msg);  // gs_capi.cu: message for gs_last_error(NULL)
}

namespace gsio {

namespace {

using u128 = unsigned __int128;

// ---- powers of ten: 10^q = F[q] * 2^B[q], F in [2^127, 2^128), F truncated ------------
constexpr int kQMin = -300, kQMax = 345;

struct Pow10Table {
    u128 f[kQMax - kQMin + 1];
    int b[kQMax - kQMin + 1];
};

// Little-endian multi-limb unsigned integer, just enough for the table.
struct Big {
    std::vector<uint64_t> w;
    int bitlen() const {
        for (int i = static_cast<int>(w.size()) - 1; i >= 0; --i)
            if (w[i]) return i * 64 + 64 - __builtin_clzll(w[i]);
        return 0;
    }
    bool bit(int i) const {
        const size_t k = static_cast<size_t>(i) / 64;
        return k < w.size() && ((w[k] >> (i % 64)) & 1u);
    }
    void mul_small(uint64_t m) {
        uint64_t carry = 0;
        for (uint64_t& x : w) {
            const u128 p = static_cast<u128>(x) * m + carry;
            x = static_cast<uint64_t>(p);
            carry = static_cast<uint64_t>(p >> 64);
        }
        if (carry) w.push_back(carry);
    }
    // top 128 bits starting at bit `lo` (bits below lo dropped)
    u128 bits_from(int lo) const {
        u128 r = 0;
        for (int i = 127; i >= 0; --i) r = (r << 1) | (bit(lo + i) ? 1u : 0u);
        return r;
    }
};

int cmp(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
    const size_t n = std::max(a.size(), b.size());
    for (size_t i = n; i-- > 0;) {
        const uint64_t x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

void sub_in_place(std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
    uint64_t borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        const uint64_t y = i < b.size() ? b[i] : 0;
        const u128 d = static_cast<u128>(a[i]) - y - borrow;
        a[i] = static_cast<uint64_t>(d);
        borrow = (d >> 64) ? 1 : 0;
    }
}

void shl1_or(std::vector<uint64_t>& a, unsigned bitv) {
    uint64_t carry = bitv;
    for (uint64_t& x : a) {
        const uint64_t nc = x >> 63;
        x = (x << 1) | carry;
        carry = nc;
    }
    if (carry) a.push_back(carry);
}

const Pow10Table& table() {
    static Pow10Table* t = [] {
        auto* tb = new Pow10Table;
        Big p;
        p.w = {1};
        // q >= 0: truncate 10^q to its top 128 bits
        for (int q = 0; q <= kQMax; ++q) {
            if (q) p.mul_small(10);
            const int L = p.bitlen();
            if (L <= 128) {
                u128 v = 0;
                for (int i = static_cast<int>(p.w.size()) - 1; i >= 0; --i) v = (v << 64) | p.w[i];
                tb->f[q - kQMin] = v << (128 - L);
                tb->b[q - kQMin] = L - 128;
            } else {
                tb->f[q - kQMin] = p.bits_from(L - 128);
                tb->b[q - kQMin] = L - 128;
            }
        }
        // q < 0: floor(2^(L+127) / 10^|q|) by binary long division (L = bitlen(10^|q|))
        Big d;
        d.w = {1};
        for (int q = 1; q <= -kQMin; ++q) {
            d.mul_small(10);
            const int L = d.bitlen();
            const int K = L + 127;
            std::vector<uint64_t> rem;
            u128 quo = 0;
            for (int i = K; i >= 0; --i) {
                shl1_or(rem, i == K ? 1u : 0u);
                quo <<= 1;
                if (cmp(rem, d.w) >= 0) {
                    sub_in_place(rem, d.w);
                    quo |= 1;
                }
            }
            tb->f[-q - kQMin] = quo;
            tb->b[-q - kQMin] = -K;
        }
        return tb;
    }();
    return *t;
}

int fallback(double v, char* out) {
    char buf[40];
    const int n = std::snprintf(buf, sizeof buf, "%.17g", v);
    std::memcpy(out, buf, static_cast<size_t>(n));
    return n;
}

constexpr uint64_t kP16 = 10000000000000000ull, kP17 = 100000000000000000ull;

}  // namespace

int fmt17(double v, char* out) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const int bexp = static_cast<int>((bits >> 52) & 0x7ff);
    const uint64_t frac = bits & ((1ull << 52) - 1);
    if (bexp == 0x7ff || (bexp == 0 && frac == 0)) return fallback(v, out);  // inf, nan, +-0
    uint64_t M;
    int e;  // |v| = M * 2^e, M in [2^63, 2^64)
    if (bexp == 0) {
        const int lz = __builtin_clzll(frac);
        M = frac << lz;
        e = -1074 - lz;
    } else {
        M = (frac | (1ull << 52)) << 11;
        e = bexp - 1075 - 11;
    }
    const int x = e + 63;                 // floor(log2 |v|)
    int e10 = (x * 78913) >> 18;          // floor(x * log10 2), |x| < 1650
    const Pow10Table& t = table();
    uint64_t N = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const int q = 16 - e10;
        const u128 F = t.f[q - kQMin];
        const u128 lo = static_cast<u128>(M) * static_cast<uint64_t>(F);
        const u128 hi = static_cast<u128>(M) * static_cast<uint64_t>(F >> 64);
        // P = hi * 2^64 + lo as three limbs w2:w1:w0
        const uint64_t w0 = static_cast<uint64_t>(lo);
        const u128 mid = (lo >> 64) + static_cast<uint64_t>(hi);
        const uint64_t w1 = static_cast<uint64_t>(mid);
        const uint64_t w2 = static_cast<uint64_t>(hi >> 64) + static_cast<uint64_t>(mid >> 64);
        const int sh = -(e + t.b[q - kQMin]);  // value * 10^q = P / 2^sh
        const int r = sh - 128;                 // 1..63 for every finite double
        if (r < 1 || r > 63) return fallback(v, out);
        const uint64_t I = w2 >> r;
        if (I >= kP17 && attempt == 0) {
            ++e10;
            continue;
        }
        // fraction = (w2 mod 2^r):w1:w0 over 2^sh; the truncated power of ten makes the
        // true fraction at most 2^64 units larger, i.e. at most +1 in the w1 limb
        const u128 fhi = (static_cast<u128>(w2 & ((1ull << r) - 1)) << 64) | w1;
        const u128 half = static_cast<u128>(1ull << (r - 1)) << 64;
        if (fhi + 2 < half) {
            N = I;
        } else if (fhi > half) {
            N = I + 1;
        } else {
            return fallback(v, out);  // within 2 ulp of a tie: let libc decide exactly
        }
        break;
    }
    if (N >= kP17) {  // rounded up across a power of ten
        N /= 10;
        ++e10;
    }
    if (N < kP16 || N >= kP17) return fallback(v, out);
    // 17 digits as 1 + 8 + 8 via 32-bit pairs
    static const char kPairs[] =
        "00010203040506070809101112131415161718192021222324252627282930313233343536373839"
        "40414243444546474849505152535455565758596061626364656667686970717273747576777879"
        "8081828384858687888990919293949596979899";
    char dig[17];
    const uint32_t top = static_cast<uint32_t>(N / 10000000000000000ull);  // 1..9
    const uint64_t rest = N - static_cast<uint64_t>(top) * 10000000000000000ull;
    uint32_t hi8 = static_cast<uint32_t>(rest / 100000000u), lo8 = static_cast<uint32_t>(rest % 100000000u);
    dig[0] = static_cast<char>('0' + top);
    for (int i = 3; i >= 0; --i) {
        std::memcpy(dig + 1 + 2 * i, kPairs + 2 * (hi8 % 100), 2);
        std::memcpy(dig + 9 + 2 * i, kPairs + 2 * (lo8 % 100), 2);
        hi8 /= 100;
        lo8 /= 100;
    }
    int nd = 17;
    while (nd > 1 && dig[nd - 1] == '0') --nd;  // %g strips trailing zeros
    char* o = out;
    if (bits >> 63) *o++ = '-';
    const int X = e10;
    if (X < -4 || X >= 17) {
        *o++ = dig[0];
        if (nd > 1) {
            *o++ = '.';
            for (int i = 1; i < nd; ++i) *o++ = dig[i];
        }
        *o++ = 'e';
        int ax = X;
        if (ax < 0) {
            *o++ = '-';
            ax = -ax;
        } else {
            *o++ = '+';
        }
        if (ax >= 100) {
            *o++ = static_cast<char>('0' + ax / 100);
            ax %= 100;
            *o++ = static_cast<char>('0' + ax / 10);
            *o++ = static_cast<char>('0' + ax % 10);
        } else {
            *o++ = static_cast<char>('0' + ax / 10);
            *o++ = static_cast<char>('0' + ax % 10);
        }
    } else if (X >= 0) {
        for (int i = 0; i <= X; ++i) *o++ = dig[i];
        if (nd > X + 1) {
            *o++ = '.';
            for (int i = X + 1; i < nd; ++i) *o++ = dig[i];
        }
    } else {
        *o++ = '0';
        *o++ = '.';
        for (int i = 0; i < -X - 1; ++i) *o++ = '0';
        for (int i = 0; i < nd; ++i) *o++ = dig[i];
    }
    return static_cast<int>(o - out);
}

void pow10_table_export(uint64_t* hi, uint64_t* lo, int* b, int* qmin, int* count) {
    const Pow10Table& t = table();
    *qmin = kQMin;
    *count = kQMax - kQMin + 1;
    for (int k = 0; k < *count; ++k) {
        hi[k] = static_cast<uint64_t>(t.f[k] >> 64);
        lo[k] = static_cast<uint64_t>(t.f[k]);
        b[k] = t.b[k];
    }
}

int default_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return static_cast<int>(std::clamp(hc ? hc : 1u, 1u, 64u));
}

namespace {

constexpr int64_t kBlock = 1 << 15;  // values per formatting block
constexpr int kMaxLen = 26;          // longest %.17g: "-1.2345678901234567e-308" + '\n'

size_t format_block(const double* u, int64_t n, char* out) {
    char* o = out;
    for (int64_t i = 0; i < n; ++i) {
        o += fmt17(u[i], o);
        *o++ = '\n';
    }
    return static_cast<size_t>(o - out);
}

// Values in order: T workers format waves of T consecutive blocks (worker i takes block
// w*T + i of wave w) into one of two buffer sets, while the calling thread writes the
// previous wave in order.  Hand-offs are two atomics per wave (no locks): a worker may start
// wave w once wave w-2 has been written, and the writer takes wave w once all T blocks of
// it are in.
bool write_values(std::FILE* f, const double* u, int64_t n, int threads) {
    const int64_t nb = (n + kBlock - 1) / kBlock;
    if (threads <= 1 || nb <= 1) {
        std::vector<char> buf(static_cast<size_t>(kBlock) * kMaxLen);
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t lo = b * kBlock, cnt = std::min(kBlock, n - lo);
            const size_t len = format_block(u + lo, cnt, buf.data());
            if (std::fwrite(buf.data(), 1, len, f) != len) return false;
        }
        return true;
    }
    const int T = static_cast<int>(std::min<int64_t>(std::min(threads, 32), nb));
    const int64_t nwaves = (nb + T - 1) / T;
    std::unique_ptr<char[]> store(new char[2 * static_cast<size_t>(T) * kBlock * kMaxLen]);  // not zeroed
    auto buf = [&](int set, int i) { return store.get() + (static_cast<size_t>(set) * T + i) * kBlock * kMaxLen; };
    std::vector<size_t> len(2 * static_cast<size_t>(T), 0);
    std::atomic<int> ready[2];
    ready[0].store(0);
    ready[1].store(0);
    std::atomic<int64_t> free_upto{2};  // waves < free_upto may be formatted
    std::atomic<bool> abort{false};
    auto worker = [&](int i) {
        for (int64_t w = 0; w < nwaves; ++w) {
            while (w >= free_upto.load(std::memory_order_acquire)) {
                if (abort.load(std::memory_order_relaxed)) return;
                std::this_thread::yield();
            }
            const int set = static_cast<int>(w & 1);
            const int64_t b = w * T + i;
            size_t l = 0;
            if (b < nb) {
                const int64_t lo = b * kBlock, cnt = std::min(kBlock, n - lo);
                l = format_block(u + lo, cnt, buf(set, i));
            }
            len[static_cast<size_t>(set) * T + i] = l;
            ready[set].fetch_add(1, std::memory_order_release);
        }
    };
    std::vector<std::thread> pool;
    for (int i = 0; i < T; ++i) pool.emplace_back(worker, i);
    bool ok = true;
    for (int64_t w = 0; w < nwaves && ok; ++w) {
        const int set = static_cast<int>(w & 1);
        while (ready[set].load(std::memory_order_acquire) < T) std::this_thread::yield();
        for (int i = 0; i < T && ok; ++i) {
            const size_t l = len[static_cast<size_t>(set) * T + i];
            if (l && std::fwrite(buf(set, i), 1, l, f) != l) ok = false;
        }
        ready[set].store(0, std::memory_order_relaxed);
        free_upto.store(w + 3, std::memory_order_release);  // wave w's set is free for wave w+2
    }
    if (!ok) abort.store(true);
    for (auto& th : pool) th.join();
    return ok;
}

}  // namespace

std::string vtk_header(int nx, int ny, int nz, double h, const double origin[3]) {
    const int64_t n = static_cast<int64_t>(nx) * ny * nz;
    char a[32], b[32], c[32];
    std::string head = "# vtk DataFile Version 3.0\ntumor density snapshot\nASCII\nDATASET STRUCTURED_POINTS\n";
    head += "DIMENSIONS " + std::to_string(nx) + ' ' + std::to_string(ny) + ' ' + std::to_string(nz) + '\n';
    const std::string hs(a, static_cast<size_t>(fmt17(h, a)));
    head += "SPACING " + hs + ' ' + hs + ' ' + hs + '\n';
    head += "ORIGIN " + std::string(a, static_cast<size_t>(fmt17(origin[0], a))) + ' ' +
            std::string(b, static_cast<size_t>(fmt17(origin[1], b))) + ' ' +
            std::string(c, static_cast<size_t>(fmt17(origin[2], c))) + '\n';
    head += "POINT_DATA " + std::to_string(n) + "\nSCALARS tumor_density float 1\nLOOKUP_TABLE default\n";
    return head;
}

bool write_vtk_stream(std::FILE* f, const std::string& path, const double* u, int nx, int ny, int nz, double h,
                      const double origin[3], const uint8_t* labels, int threads, Error& err) {
    const int64_t n = static_cast<int64_t>(nx) * ny * nz;
    const std::string head = vtk_header(nx, ny, nz, h, origin);
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    ok = ok && write_values(f, u, n, threads <= 0 ? default_threads() : threads);
    if (ok && labels) {
        static const char kHead[] = "SCALARS material int 1\nLOOKUP_TABLE default\n";
        ok = std::fwrite(kHead, 1, sizeof kHead - 1, f) == sizeof kHead - 1;
        constexpr int64_t kChunk = 1 << 20;
        std::vector<char> buf(4 * static_cast<size_t>(std::min<int64_t>(n, kChunk)));  // "255\n" at most
        for (int64_t lo = 0; ok && lo < n; lo += kChunk) {
            const int64_t cnt = std::min<int64_t>(n - lo, kChunk);
            size_t l = 0;
            for (int64_t i = 0; i < cnt; ++i) {
                // Material codes are printed as int (vtk.cpp:85)
                const int code = labels[lo + i];
                if (code >= 100) buf[l++] = static_cast<char>('0' + code / 100);
                if (code >= 10) buf[l++] = static_cast<char>('0' + (code / 10) % 10);
                buf[l++] = static_cast<char>('0' + code % 10);
                buf[l++] = '\n';
            }
            if (std::fwrite(buf.data(), 1, l, f) != l) ok = false;
        }
    }
    if (ok && std::fflush(f) != 0) ok = false;
    if (!ok) {
        err.code = GS_EDATA;
        err.msg = "write failed: " + path;
    }
    return ok;
}

namespace {

// ---- read_vtk ------------------------------------------------------------------------
inline bool is_space(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

struct Reader {
    const char* p;
    const char* end;
    const std::string& path;
    Error& err;

    bool token(std::string& tok) {
        while (p < end && is_space(static_cast<unsigned char>(*p))) ++p;
        if (p == end) {
            err = {GS_EDATA, path + ": unexpected end of file"};
            return false;
        }
        const char* s = p;
        while (p < end && !is_space(static_cast<unsigned char>(*p))) ++p;
        tok.assign(s, p);
        return true;
    }
    bool expect(const char* want) {
        std::string tok;
        if (!token(tok)) return false;
        if (tok != want) {
            err = {GS_EDATA, path + ": expected '" + want + "', found '" + tok + "'"};
            return false;
        }
        return true;
    }
    // std::stoi semantics (strtol, int range, whole token) plus v >= 1 (vtk.cpp:34-45)
    bool count(int& v) {
        std::string tok;
        if (!token(tok)) return false;
        errno = 0;
        char* e = nullptr;
        const long x = std::strtol(tok.c_str(), &e, 10);
        if (e == tok.c_str() || errno == ERANGE || x < INT_MIN || x > INT_MAX ||
            static_cast<size_t>(e - tok.c_str()) != tok.size() || x < 1) {
            err = {GS_EDATA, path + ": expected a positive integer, found '" + tok + "'"};
            return false;
        }
        v = static_cast<int>(x);
        return true;
    }
    bool value(double& v) {
        std::string tok;
        if (!token(tok)) return false;
        return parse_double(tok.c_str(), tok.size(), v) || bad_number(tok);
    }
    bool bad_number(const std::string& tok) {
        err = {GS_EDATA, path + ": expected a number, found '" + tok + "'"};
        return false;
    }
    // std::stod semantics (vtk.cpp:47-57): strtod, ERANGE rejected, whole token
    static bool parse_double(const char* s, size_t len, double& v) {
        errno = 0;
        char* e = nullptr;
        const double x = std::strtod(s, &e);
        if (e == s || errno == ERANGE || static_cast<size_t>(e - s) != len) return false;
        v = x;
        return true;
    }
};

struct Chunk {
    std::vector<double> vals;
    bool bad = false;
    std::string bad_tok;
};

// Parses every whitespace-separated token of [s, e) as a double until the first failure.
void parse_chunk(const char* s, const char* e, Chunk& c) {
    char small[64];
    while (s < e) {
        while (s < e && is_space(static_cast<unsigned char>(*s))) ++s;
        if (s == e) break;
        const char* t = s;
        while (s < e && !is_space(static_cast<unsigned char>(*s))) ++s;
        const size_t len = static_cast<size_t>(s - t);
        double v;
        bool ok;
        if (len < sizeof small) {
            std::memcpy(small, t, len);
            small[len] = 0;
            ok = Reader::parse_double(small, len, v);
        } else {
            const std::string tok(t, len);
            ok = Reader::parse_double(tok.c_str(), len, v);
        }
        if (!ok) {
            c.bad = true;
            c.bad_tok.assign(t, len);
            return;
        }
        c.vals.push_back(v);
    }
}

bool slurp(const char* path, std::string& data) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    char buf[1 << 16];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) data.append(buf, k);
    std::fclose(f);
    return true;
}

gs_status fail_free(gs_status code, const std::string& msg) {
    set_free_error(msg);
    return code;
}

gs_status fail_free(const Error& e) { return fail_free(static_cast<gs_status>(e.code), e.msg); }

// std::getline: true when at least one character or a '\n' was extracted
bool get_line(const std::string& d, size_t& pos, std::string& line) {
    if (pos >= d.size()) return false;
    const size_t nl = d.find('\n', pos);
    if (nl == std::string::npos) {
        line = d.substr(pos);
        pos = d.size();
    } else {
        line = d.substr(pos, nl - pos);
        pos = nl + 1;
    }
    return true;
}

// ---- PGM (imaging.cpp:14-61) -----------------------------------------------------------
struct PgmIn {
    const std::string& d;
    size_t pos = 0;
    const std::string& path;
    Error& err;

    bool token(std::string& tok) {
        while (pos < d.size()) {
            const unsigned char c = static_cast<unsigned char>(d[pos++]);
            if (c == '#') {
                while (pos < d.size() && d[pos++] != '\n') {}
                continue;
            }
            if (is_space(c)) continue;
            tok.assign(1, static_cast<char>(c));
            while (pos < d.size() && !is_space(static_cast<unsigned char>(d[pos])) && d[pos] != '#')
                tok.push_back(d[pos++]);
            return true;
        }
        err = {GS_EDATA, "pgm: '" + path + "': truncated header"};
        return false;
    }
    bool integer(const char* what, int& v) {
        std::string tok;
        if (!token(tok)) return false;
        errno = 0;
        char* e = nullptr;
        const long x = std::strtol(tok.c_str(), &e, 10);
        if (e == tok.c_str() || errno == ERANGE || x < INT_MIN || x > INT_MAX ||
            static_cast<size_t>(e - tok.c_str()) != tok.size() || x < 0) {
            err = {GS_EDATA, "pgm: '" + path + "': bad " + what + " '" + tok + "'"};
            return false;
        }
        v = static_cast<int>(x);
        return true;
    }
};

// One slice: validates like load_pgm and returns the offset/size of its pixel bytes.
bool load_pgm(const std::string& path, std::string& data, int& w, int& h, size_t& pix, Error& err) {
    data.clear();
    if (!slurp(path.c_str(), data)) {
        err = {GS_EDATA, "pgm: cannot open '" + path + "'"};
        return false;
    }
    PgmIn in{data, 0, path, err};
    std::string magic;
    if (!in.token(magic)) return false;
    if (magic != "P5") {
        err = {GS_EDATA, "pgm: '" + path + "': magic is '" + magic + "', expected P5"};
        return false;
    }
    int maxval = 0;
    if (!in.integer("width", w) || !in.integer("height", h) || !in.integer("maxval", maxval)) return false;
    if (maxval != 255) {
        err = {GS_EDATA, "pgm: '" + path + "': maxval " + std::to_string(maxval) + ", expected 255"};
        return false;
    }
    if (in.pos < data.size()) ++in.pos;  // the single whitespace byte after maxval
    const size_t n = static_cast<size_t>(w) * static_cast<size_t>(h);
    if (data.size() - in.pos < n) {
        err = {GS_EDATA, "pgm: '" + path + "': truncated pixel data"};
        return false;
    }
    pix = in.pos;
    return true;
}

// ---- raw volume (imaging.cpp:95-116) ---------------------------------------------------
bool load_raw(const char* path_c, std::string& data, int& w, int& h, int& s, size_t& pix, Error& err) {
    const std::string path(path_c);
    if (!slurp(path_c, data)) {
        err = {GS_EDATA, "raw volume: cannot open '" + path + "'"};
        return false;
    }
    size_t pos = 0;
    std::string header;
    if (!get_line(data, pos, header)) {
        err = {GS_EDATA, "raw volume: '" + path + "': missing header"};
        return false;
    }
    std::istringstream hs(header);
    if (!(hs >> w >> h >> s) || w < 1 || h < 1 || s < 1) {
        err = {GS_EDATA, "raw volume: '" + path + "': bad header '" + header + "'"};
        return false;
    }
    std::string rest;
    if (hs >> rest) {
        err = {GS_EDATA, "raw volume: '" + path + "': trailing header token '" + rest + "'"};
        return false;
    }
    const size_t n = static_cast<size_t>(w) * static_cast<size_t>(h) * static_cast<size_t>(s);
    if (data.size() - pos < n) {
        err = {GS_EDATA, "raw volume: '" + path + "': truncated voxel data"};
        return false;
    }
    pix = pos;
    return true;
}

}  // namespace

}  // namespace gsio

using gsio::Error;

extern "C" {

gs_status gs_write_vtk(const char* path, const double* u, int nx, int ny, int nz, double h, const double origin[3],
                       const uint8_t* labels, int threads) {
    if (!path || !u || !origin) return gsio::fail_free(GS_EINVAL, "write_vtk: null argument");
    if (nx < 1 || ny < 1 || nz < 1) return gsio::fail_free(GS_EINVAL, "Grid: point counts must be >= 1");
    if (!(h > 0.0)) return gsio::fail_free(GS_EINVAL, "Grid: spacing h must be positive");
    std::FILE* f = std::fopen(path, "w");
    if (!f) return gsio::fail_free(GS_EDATA, std::string("cannot open ") + path + " for writing");
    Error err;
    const bool ok = gsio::write_vtk_stream(f, path, u, nx, ny, nz, h, origin, labels, threads, err);
    const bool closed = std::fclose(f) == 0;
    if (!ok) return gsio::fail_free(err);
    if (!closed) return gsio::fail_free(GS_EDATA, std::string("write failed: ") + path);
    return GS_OK;
}

gs_status gs_read_vtk(const char* path_c, int dims[3], double* h, double origin[3], double* values,
                      int64_t capacity, int threads) {
    if (!path_c || !dims || !h || !origin) return gsio::fail_free(GS_EINVAL, "read_vtk: null argument");
    const std::string path(path_c);
    std::string data;
    if (!gsio::slurp(path_c, data)) return gsio::fail_free(GS_EDATA, "cannot open " + path);
    size_t pos = 0;
    std::string line;
    if (!gsio::get_line(data, pos, line) || line.rfind("# vtk DataFile", 0) != 0)
        return gsio::fail_free(GS_EDATA, path + ": missing '# vtk DataFile' header");
    if (!gsio::get_line(data, pos, line)) return gsio::fail_free(GS_EDATA, path + ": missing title line");
    Error err;
    gsio::Reader r{data.data() + pos, data.data() + data.size(), path, err};
    int nx = 0, ny = 0, nz = 0, n = 0;
    double hx = 0, hy = 0, hz = 0, o[3] = {0, 0, 0};
    std::string skip;
    bool ok = r.expect("ASCII") && r.expect("DATASET") && r.expect("STRUCTURED_POINTS") && r.expect("DIMENSIONS") &&
              r.count(nx) && r.count(ny) && r.count(nz) && r.expect("SPACING") && r.value(hx) && r.value(hy) &&
              r.value(hz);
    if (!ok) return gsio::fail_free(err);
    if (!(hx > 0.0) || hx != hy || hy != hz)
        return gsio::fail_free(GS_EDATA, path + ": spacing must be positive and isotropic");
    ok = r.expect("ORIGIN") && r.value(o[0]) && r.value(o[1]) && r.value(o[2]) && r.expect("POINT_DATA") && r.count(n);
    if (!ok) return gsio::fail_free(err);
    if (static_cast<int64_t>(n) != static_cast<int64_t>(nx) * ny * nz)
        return gsio::fail_free(GS_EDATA, path + ": POINT_DATA count disagrees with DIMENSIONS");
    ok = r.expect("SCALARS") && r.expect("tumor_density") && r.token(skip) && r.token(skip) &&
         r.expect("LOOKUP_TABLE") && r.token(skip);
    if (!ok) return gsio::fail_free(err);
    dims[0] = nx;
    dims[1] = ny;
    dims[2] = nz;
    *h = hx;
    origin[0] = o[0];
    origin[1] = o[1];
    origin[2] = o[2];
    if (!values) return GS_OK;  // header only
    if (capacity < n) return gsio::fail_free(GS_EINVAL, "read_vtk: value buffer too small");

    // Values: split the rest of the file into chunks at whitespace, parse them in parallel,
    // then take the first n tokens in order (anything after them -- the material array --
    // is ignored, as in the reference).
    const char* s = r.p;
    const char* e = r.end;
    const int T = std::max(1, std::min(threads <= 0 ? gsio::default_threads() : threads,
                                       static_cast<int>((e - s) / (1 << 20)) + 1));
    std::vector<const char*> cut(static_cast<size_t>(T) + 1, e);
    cut[0] = s;
    for (int i = 1; i < T; ++i) {
        const char* c = std::max(cut[i - 1], s + (e - s) * i / T);
        while (c < e && !gsio::is_space(static_cast<unsigned char>(*c))) ++c;
        cut[i] = c;
    }
    std::vector<gsio::Chunk> chunks(static_cast<size_t>(T));
    if (T == 1) {
        gsio::parse_chunk(s, e, chunks[0]);
    } else {
        std::vector<std::thread> pool;
        for (int i = 0; i < T; ++i)
            pool.emplace_back([&, i] { gsio::parse_chunk(cut[i], cut[i + 1], chunks[i]); });
        for (auto& th : pool) th.join();
    }
    int64_t got = 0;
    for (const gsio::Chunk& c : chunks) {
        const int64_t take = std::min<int64_t>(static_cast<int64_t>(c.vals.size()), n - got);
        std::memcpy(values + got, c.vals.data(), static_cast<size_t>(take) * sizeof(double));
        got += take;
        if (got == n) return GS_OK;
        if (c.bad) return gsio::fail_free(GS_EDATA, path + ": expected a number, found '" + c.bad_tok + "'");
    }
    return gsio::fail_free(GS_EDATA, path + ": unexpected end of file");
}

gs_status gs_write_metrics_csv(const char* path, int count, const int32_t* step, const double* time,
                               const gs_metrics* m) {
    if (!path || count < 0 || (count > 0 && (!step || !time || !m)))
        return gsio::fail_free(GS_EINVAL, "write_metrics_csv: null argument");
    std::FILE* f = std::fopen(path, "w");
    if (!f) return gsio::fail_free(GS_EDATA, std::string("cannot open ") + path + " for writing");
    std::string out = "step,time_days,total_mass,max_density,radius_mm\n";
    char b[32];
    for (int i = 0; i < count; ++i) {
        out += std::to_string(step[i]);
        const double cols[4] = {time[i], m[i].total_mass, m[i].max_density, m[i].radius};
        for (double v : cols) {
            out += ',';
            out.append(b, static_cast<size_t>(gsio::fmt17(v, b)));
        }
        out += '\n';
    }
    const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
    const bool closed = std::fclose(f) == 0;
    if (!ok || !closed) return gsio::fail_free(GS_EDATA, std::string("write failed: ") + path);
    return GS_OK;
}

gs_status gs_load_stack(const char* const* paths, int count, int* width, int* height, int* slices, uint8_t* out,
                        int64_t capacity) {
    if (!width || !height || !slices) return gsio::fail_free(GS_EINVAL, "load_stack: null argument");
    if (count <= 0 || !paths) return gsio::fail_free(GS_EDATA, "load_stack: no slice files given");
    std::string data;
    int W = 0, H = 0;
    int64_t off = 0;
    for (int i = 0; i < count; ++i) {
        const std::string path(paths[i] ? paths[i] : "");
        int w = 0, h = 0;
        size_t pix = 0;
        Error err;
        if (!gsio::load_pgm(path, data, w, h, pix, err)) return gsio::fail_free(err);
        if (i == 0) {
            W = w;
            H = h;
        } else if (w != W || h != H) {
            return gsio::fail_free(GS_EDATA, "load_stack: '" + path + "' is " + std::to_string(w) + "x" +
                                                 std::to_string(h) + ", previous slices are " + std::to_string(W) +
                                                 "x" + std::to_string(H));
        }
        const int64_t n = static_cast<int64_t>(w) * h;
        if (out) {
            if (off + n > capacity) return gsio::fail_free(GS_EINVAL, "load_stack: output buffer too small");
            std::memcpy(out + off, data.data() + pix, static_cast<size_t>(n));
        }
        off += n;
    }
    *width = W;
    *height = H;
    *slices = count;
    return GS_OK;
}

gs_status gs_load_raw_volume(const char* path, int* width, int* height, int* slices, uint8_t* out,
                             int64_t capacity) {
    if (!path || !width || !height || !slices) return gsio::fail_free(GS_EINVAL, "load_raw_volume: null argument");
    std::string data;
    int w = 0, h = 0, s = 0;
    size_t pix = 0;
    Error err;
    if (!gsio::load_raw(path, data, w, h, s, pix, err)) return gsio::fail_free(err);
    const int64_t n = static_cast<int64_t>(w) * h * s;
    if (out) {
        if (capacity < n) return gsio::fail_free(GS_EINVAL, "load_raw_volume: output buffer too small");
        std::memcpy(out, data.data() + pix, static_cast<size_t>(n));
    }
    *width = w;
    *height = h;
    *slices = s;
    return GS_OK;
}

gs_status gs_write_label_volume(const char* path, const uint8_t* labels, int nx, int ny, int nz) {
    if (!path || !labels) return gsio::fail_free(GS_EINVAL, "write_label_volume: null argument");
    if (nx < 1 || ny < 1 || nz < 1) return gsio::fail_free(GS_EINVAL, "Grid: point counts must be >= 1");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return gsio::fail_free(GS_EDATA, std::string("label volume: cannot open '") + path + "'");
    const std::string head = std::to_string(nx) + ' ' + std::to_string(ny) + ' ' + std::to_string(nz) + '\n';
    const size_t n = static_cast<size_t>(nx) * static_cast<size_t>(ny) * static_cast<size_t>(nz);
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    ok = ok && std::fwrite(labels, 1, n, f) == n;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return gsio::fail_free(GS_EDATA, std::string("label volume: write failure on '") + path + "'");
    return GS_OK;
}

gs_status gs_read_label_volume(const char* path, int nx, int ny, int nz, uint8_t* labels) {
    if (!path || !labels) return gsio::fail_free(GS_EINVAL, "read_label_volume: null argument");
    if (nx < 1 || ny < 1 || nz < 1) return gsio::fail_free(GS_EINVAL, "Grid: point counts must be >= 1");
    std::string data;
    int w = 0, h = 0, s = 0;
    size_t pix = 0;
    Error err;
    if (!gsio::load_raw(path, data, w, h, s, pix, err)) return gsio::fail_free(err);
    if (w != nx || h != ny || s != nz)
        return gsio::fail_free(GS_EDATA, std::string("label volume: '") + path + "' is " + std::to_string(w) + "x" +
                                             std::to_string(h) + "x" + std::to_string(s) + ", grid wants " +
                                             std::to_string(nx) + "x" + std::to_string(ny) + "x" +
                                             std::to_string(nz));
    const size_t n = static_cast<size_t>(w) * static_cast<size_t>(h) * static_cast<size_t>(s);
    const auto* src = reinterpret_cast<const uint8_t*>(data.data() + pix);
    for (size_t v = 0; v < n; ++v)
        if (src[v] > 3)
            return gsio::fail_free(GS_EDATA, std::string("label volume: '") + path + "': byte " +
                                                 std::to_string(src[v]) + " is not a material label");
    std::memcpy(labels, src, n);
    return GS_OK;
}

}  // extern "C"
