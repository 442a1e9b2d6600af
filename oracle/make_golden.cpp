// make_golden.cpp — writes tests/golden/*.json from the REFERENCE itself.
//
// Replays the reference's own seeded suites (same seeds, same draw order) with
// the reference's generators/encoders (tests/support/oracles.hpp, included in
// place from /root/reference) and records the outputs of the reference CPU
// harness (interp::register_reference_harnesses, src/interp.cpp:330-389).
// Build + run: `make -C oracle golden` (needs /root/reference; test infra only).

#include "lilac/how.hpp"
#include "lilac/interp.hpp"
#include "lilac/marshal.hpp"
#include "lilac/what.hpp"
#include "support/oracles.hpp"
#include "support/programs.hpp"

#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

using namespace lilac;

namespace {

std::string num(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

template <typename T>
std::string arr(const std::vector<T>& v) {
    std::ostringstream os;
    os << "[";
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) os << ",";
        if constexpr (std::is_floating_point_v<T>)
            os << num(v[i]);
        else
            os << v[i];
    }
    os << "]";
    return os.str();
}

interp::HarnessRegistry& reg() {
    static interp::HarnessRegistry r = [] {
        interp::HarnessRegistry h;
        std::vector<what::WhatProgram> ps;
        ps.push_back(what::parse_what(programs::kSpmvCsr));
        ps.push_back(what::parse_what(programs::kSpmvJds));
        ps.push_back(what::parse_what(programs::kDotProduct));
        ps.push_back(what::parse_what(programs::kGemm));
        interp::register_reference_harnesses(h, ps);
        return h;
    }();
    return r;
}

std::vector<double> ref_csr(const oracle::Csr& m, const std::vector<double>& xv) {
    interp::Memory mem;
    int out = mem.alloc_floats("output", std::vector<double>(static_cast<size_t>(m.rows), 0.0));
    int rp = mem.alloc_ints("row_ptr", m.row_ptr);
    int v = mem.alloc_floats("val", m.val);
    int x = mem.alloc_floats("x", xv);
    int ci = mem.alloc_ints("col_ind", m.col_ind);
    std::vector<interp::Value> args = {m.rows, interp::Pointer{out, 0}, interp::Pointer{rp, 0},
                                       interp::Pointer{v, 0}, interp::Pointer{x, 0},
                                       interp::Pointer{ci, 0}};
    (*reg().find("lilac.spmv_csr"))(mem, args);
    return mem.floats(out);
}

std::vector<double> ref_jds(const oracle::Jds& m, const std::vector<double>& xv) {
    interp::Memory mem;
    int out = mem.alloc_floats("output", std::vector<double>(static_cast<size_t>(m.rows), 0.0));
    int nz = mem.alloc_ints("nzcnt", m.nzcnt);
    int pm = mem.alloc_ints("perm", m.perm);
    int v = mem.alloc_floats("val", m.val);
    int jd = mem.alloc_ints("jd_ptr", m.jd_ptr);
    int x = mem.alloc_floats("x", xv);
    int ci = mem.alloc_ints("col_ind", m.col_ind);
    std::vector<interp::Value> args = {m.rows,
                                       interp::Pointer{out, 0},
                                       interp::Pointer{nz, 0},
                                       interp::Pointer{pm, 0},
                                       interp::Pointer{v, 0},
                                       interp::Pointer{jd, 0},
                                       interp::Pointer{x, 0},
                                       interp::Pointer{ci, 0}};
    (*reg().find("lilac.spmv_jds"))(mem, args);
    return mem.floats(out);
}

std::vector<double> ref_gemm(std::int64_t n, std::int64_t m, std::int64_t p, const std::vector<double>& av,
                             const std::vector<double>& bv) {
    interp::Memory mem;
    int c = mem.alloc_floats("c", std::vector<double>(static_cast<size_t>(n * m), 0.0));
    int a = mem.alloc_floats("a", av);
    int b = mem.alloc_floats("b", bv);
    std::vector<interp::Value> args = {n, m, interp::Pointer{c, 0}, p, interp::Pointer{a, 0}, interp::Pointer{b, 0}};
    (*reg().find("lilac.gemm"))(mem, args);
    return mem.floats(c);
}

double ref_dot(const std::vector<double>& av, const std::vector<double>& bv) {
    interp::Memory mem;
    int a = mem.alloc_floats("a", av);
    int b = mem.alloc_floats("b", bv);
    std::vector<interp::Value> args = {static_cast<std::int64_t>(av.size()), interp::Pointer{a, 0},
                                       interp::Pointer{b, 0}};
    return std::get<double>((*reg().find("lilac.dotproduct"))(mem, args));
}

std::string case_json(int64_t rows, int64_t cols, const std::vector<double>& dense,
                      const std::vector<double>& x) {
    oracle::Csr c = oracle::csr_from_dense(rows, cols, dense);
    oracle::Jds j = oracle::jds_from_dense(rows, cols, dense);
    std::vector<double> yc = ref_csr(c, x);
    std::vector<double> yj = ref_jds(j, x);
    std::ostringstream os;
    os << "{\"rows\":" << rows << ",\"cols\":" << cols << ",\"dense\":" << arr(dense)
       << ",\"x\":" << arr(x) << ",\"csr\":{\"row_ptr\":" << arr(c.row_ptr)
       << ",\"col_ind\":" << arr(c.col_ind) << ",\"val\":" << arr(c.val) << "}"
       << ",\"jds\":{\"perm\":" << arr(j.perm) << ",\"nzcnt\":" << arr(j.nzcnt)
       << ",\"jd_ptr\":" << arr(j.jd_ptr) << ",\"col_ind\":" << arr(j.col_ind)
       << ",\"val\":" << arr(j.val) << "}"
       << ",\"y_csr\":" << arr(yc) << ",\"y_jds\":" << arr(yj)
       << ",\"y_dense\":" << arr(oracle::dense_spmv(rows, cols, dense, x)) << "}";
    return os.str();
}

void write(const std::string& path, const std::string& body) {
    std::ofstream f(path);
    f << body << "\n";
}

std::string sig_of(const char* text) {
    what::HarnessSignature s = what::infer_interface(what::parse_what(text));
    std::string r = "[";
    for (size_t i = 0; i < s.params.size(); ++i) {
        if (i) r += ",";
        r += "[\"" + s.params[i].name + "\",\"" + what::param_kind_name(s.params[i].kind) + "\"]";
    }
    return r + "]";
}

} // namespace

int main(int argc, char** argv) {
    std::string dir = argc > 1 ? argv[1] : "tests/golden";

    // sample5 (oracles.hpp:186-213; fixtures/data/sample5_*.json)
    {
        using namespace oracle::sample5;
        std::ostringstream os;
        os << "{\"source\":\"tests/support/oracles.hpp:186-213 via lilac.spmv_csr/spmv_jds\","
           << "\"ones\":" << case_json(rows, cols, dense, oracle::ones(5))
           << ",\"counting\":" << case_json(rows, cols, dense, {1, 2, 3, 4, 5})
           << ",\"frozen\":{\"csr_val\":" << arr(csr_val) << ",\"csr_col_ind\":" << arr(csr_col_ind)
           << ",\"csr_row_ptr\":" << arr(csr_row_ptr) << ",\"jds_perm\":" << arr(jds_perm)
           << ",\"jds_jd_ptr\":" << arr(jds_jd_ptr) << ",\"jds_val\":" << arr(jds_val)
           << ",\"jds_col_ind\":" << arr(jds_col_ind) << ",\"jds_nzcnt\":" << arr(jds_nzcnt)
           << ",\"y_ones\":" << arr(y_ones) << ",\"y_counting\":" << arr(y_counting) << "}}";
        write(dir + "/sample5.json", os.str());
    }

    // test_what.cpp:84-95 — seed 20240817, 50 trials, n in [1,16], density 0.3
    {
        std::mt19937_64 rng(20240817);
        std::ostringstream os;
        os << "{\"source\":\"tests/test_what.cpp:84-95 (seed 20240817)\",\"cases\":[";
        for (int t = 0; t < 50; ++t) {
            std::int64_t n = 1 + static_cast<std::int64_t>(rng() % 16);
            std::vector<double> dense = oracle::random_dense(rng, n, n, 0.3);
            std::vector<double> x = oracle::random_vector(rng, n);
            os << (t ? "," : "") << case_json(n, n, dense, x);
        }
        os << "]}";
        write(dir + "/what_csr_seed20240817.json", os.str());
    }

    // test_what.cpp:97-114 — seed 7, 20 trials, n in [1,12], density 0.4
    {
        std::mt19937_64 rng(7);
        std::ostringstream os;
        os << "{\"source\":\"tests/test_what.cpp:97-114 (seed 7)\",\"cases\":[";
        for (int t = 0; t < 20; ++t) {
            std::int64_t n = 1 + static_cast<std::int64_t>(rng() % 12);
            std::vector<double> dense = oracle::random_dense(rng, n, n, 0.4);
            std::vector<double> x = oracle::random_vector(rng, n);
            os << (t ? "," : "") << case_json(n, n, dense, x);
        }
        os << "]}";
        write(dir + "/what_jds_seed7.json", os.str());
    }

    // test_interp.cpp:215-300 — seed 424242, 50 trials, rectangular, density 0.4;
    // each case also carries the gemm harness call of the same trial
    // (n = rows, m = cols, a = random_dense(n, p), b = random_dense(p, m)).
    {
        std::mt19937_64 rng(424242);
        std::ostringstream os;
        os << "{\"source\":\"tests/test_interp.cpp:215-300 (seed 424242)\",\"cases\":[";
        for (int t = 0; t < 50; ++t) {
            std::int64_t rows = 1 + static_cast<std::int64_t>(rng() % 8);
            std::int64_t cols = 1 + static_cast<std::int64_t>(rng() % 8);
            std::vector<double> dense = oracle::random_dense(rng, rows, cols, 0.4);
            std::vector<double> x = oracle::random_vector(rng, cols);
            std::string cj = case_json(rows, cols, dense, x);
            std::int64_t p = 1 + static_cast<std::int64_t>(rng() % 6);
            std::vector<double> ga = oracle::random_dense(rng, rows, p, 0.8);
            std::vector<double> gb = oracle::random_dense(rng, p, cols, 0.8);
            std::ostringstream g;
            g << ",\"gemm\":{\"n\":" << rows << ",\"m\":" << cols << ",\"p\":" << p << ",\"a\":" << arr(ga)
              << ",\"b\":" << arr(gb) << ",\"c\":" << arr(ref_gemm(rows, cols, p, ga, gb)) << "}}";
            cj.back() == '}' ? cj.pop_back() : void();
            os << (t ? "," : "") << cj << g.str();
        }
        os << "]}";
        write(dir + "/interp_harness_seed424242.json", os.str());
    }

    // test_interp.cpp:188-213 — dot, seed 5150, 20 trials, n in [0,8]
    {
        std::mt19937_64 rng(5150);
        std::ostringstream os;
        os << "{\"source\":\"tests/test_interp.cpp:188-213 (seed 5150)\",\"cases\":[";
        for (int t = 0; t < 20; ++t) {
            std::int64_t n = static_cast<std::int64_t>(rng() % 9);
            std::vector<double> a = oracle::random_vector(rng, n);
            std::vector<double> b = oracle::random_vector(rng, n);
            os << (t ? "," : "") << "{\"a\":" << arr(a) << ",\"b\":" << arr(b)
               << ",\"result\":" << num(ref_dot(a, b)) << ",\"oracle_dot\":" << num(oracle::dot(a, b))
               << "}";
        }
        os << "]}";
        write(dir + "/dot_seed5150.json", os.str());
    }

    // marshal: FNV-1a vectors (test_marshal.cpp:30-34) and harness signatures
    // (test_what.cpp:164-201, what_parse.cpp:356-429).
    {
        std::ostringstream os;
        os << "{\"source\":\"tests/test_marshal.cpp:30-34; tests/test_what.cpp:164-201\","
           << "\"fnv1a\":[[\"\"," << marshal::fnv1a("", 0) << "],[\"a\"," << marshal::fnv1a("a", 1)
           << "],[\"foobar\"," << marshal::fnv1a("foobar", 6) << "]],"
           << "\"signatures\":{\"spmv_csr\":" << sig_of(programs::kSpmvCsr)
           << ",\"spmv_jds\":" << sig_of(programs::kSpmvJds)
           << ",\"dotproduct\":" << sig_of(programs::kDotProduct)
           << ",\"gemm\":" << sig_of(programs::kGemm) << "}}";
        write(dir + "/abi.json", os.str());
    }
    std::printf("golden fixtures written to %s\n", dir.c_str());
    return 0;
}
