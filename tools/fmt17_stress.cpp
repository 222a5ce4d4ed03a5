// Stress check of gsio::fmt17 against glibc snprintf("%.17g") (the reference's vtk.cpp:16-20).
//   g++ -O2 -std=c++17 -I include -I paper_2402_02273_b200/csrc tools/fmt17_stress.cpp -o /tmp/fmt17 -lpthread
//   /tmp/fmt17 [millions]
#include "../paper_2402_02273_b200/csrc/gs_io.cpp"

#include <chrono>
#include <cmath>
#include <random>

namespace gsio {
void set_free_error(const std::string&) {}
}

int main(int argc, char** argv) {
    const long millions = argc > 1 ? std::atol(argv[1]) : 20;
    std::mt19937_64 rng(12345);
    long bad = 0, total = 0;
    auto check = [&](double v) {
        char a[40], b[40];
        const int n = gsio::fmt17(v, a);
        a[n] = 0;
        std::snprintf(b, sizeof b, "%.17g", v);
        ++total;
        if (std::strcmp(a, b) != 0 && bad++ < 20) std::printf("MISMATCH %a: got %s want %s\n", v, a, b);
    };
    // structured cases
    for (int e = -1074; e <= 1023; ++e) {
        const double p = std::ldexp(1.0, e);
        check(p);
        check(-p);
        check(std::nextafter(p, 0.0));
        check(std::nextafter(p, INFINITY));
    }
    for (int k = -330; k <= 310; ++k) {
        const double p = std::pow(10.0, k);
        for (double q : {p, std::nextafter(p, 0.0), std::nextafter(p, INFINITY), 5 * p, 9.9999999999999995 * p})
            if (std::isfinite(q)) check(q);
    }
    for (long i = 0; i < 1000000; ++i) check(static_cast<double>(i));
    for (long i = 0; i < 1000000; ++i) check(i / 1024.0);
    const double specials[] = {0.0, -0.0, INFINITY, -INFINITY, NAN, 1.0 / 3, 0.1, 1e-17, 4.9406564584124654e-324,
                               2.2250738585072014e-308, 1.7976931348623157e308, 123456789012345678.0};
    for (double v : specials) check(v);
    // random bit patterns and uniform values
    const auto t0 = std::chrono::steady_clock::now();
    for (long i = 0; i < millions * 1000000; ++i) {
        uint64_t bits = rng();
        double v;
        std::memcpy(&v, &bits, 8);
        if (i & 1) v = std::uniform_real_distribution<double>(0.0, 1.0)(rng);
        check(v);
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // throughput of fmt17 alone
    std::vector<double> xs(4000000);
    for (double& x : xs) x = std::uniform_real_distribution<double>(0.0, 1.0)(rng) * (rng() % 3 ? 1 : 1e-7);
    char buf[40];
    size_t sink = 0;
    auto t1 = std::chrono::steady_clock::now();
    for (double x : xs) sink += gsio::fmt17(x, buf);
    const double f_ns = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count() / xs.size() * 1e9;
    t1 = std::chrono::steady_clock::now();
    for (double x : xs) sink += std::snprintf(buf, sizeof buf, "%.17g", x);
    const double s_ns = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count() / xs.size() * 1e9;
    std::printf("checked %ld values (%.1f s), mismatches %ld; fmt17 %.1f ns/value, snprintf %.1f ns/value (%zu)\n",
                total, secs, bad, f_ns, s_ns, sink);
    return bad != 0;
}
