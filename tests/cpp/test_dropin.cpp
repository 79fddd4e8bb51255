// Drop-in check: code written against the reference API (namespace fftmv,
// reference headers' names and signatures) compiles unchanged against
// include/fftmv/*.hpp and runs on the B200 kernels.
//   build/fftmv_cpp_tests          host-only checks (no GPU needed)
//   build/fftmv_cpp_tests --gpu    + operator setup / matvecs / partition / sweep on cuda:0
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fftmv/block_vector.hpp"
#include "fftmv/config.hpp"
#include "fftmv/dims.hpp"
#include "fftmv/fft.hpp"
#include "fftmv/gemv.hpp"
#include "fftmv/matvec.hpp"
#include "fftmv/operator.hpp"
#include "fftmv/partition.hpp"
#include "fftmv/random_fill.hpp"
#include "fftmv/sweep.hpp"
#include "fftmv/vector_io.hpp"

using namespace fftmv;

static int failures = 0;
#define EXPECT(c)                                                          \
  do {                                                                     \
    if (!(c)) {                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);             \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <class F>
static bool throws_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  }
  return false;
}

static void host_checks() {
  EXPECT(throws_invalid([] { ProblemDims(0, 1, 1); }));
  EXPECT(ProblemDims(5, 3, 7).fft_len() == 14 && ProblemDims(5, 3, 7).n_bins() == 8);
  EXPECT(parse_precision_config("dssdd").render() == "dssdd");
  EXPECT(throws_invalid([] { parse_precision_config("dsxdd"); }));
  EXPECT(parse_precision_config("ddmdd").render() == "ddmdd");  // fp32 storage, fp64 accumulation (slot 3 only)
  EXPECT(parse_precision_config("ddmdd")[2] == Precision::SingleAccDouble);
  EXPECT(throws_invalid([] { parse_precision_config("dmddd"); }));
  EXPECT(throws_invalid([] { parse_precision_config("dss"); }));
  auto all = enumerate_configs();
  EXPECT(all.size() == 32 && all.front().render() == "ddddd" && all.back().render() == "sssss");
  EXPECT(all[1].render() == "dddds");
  auto g = Grid1xP::split(3, 5);
  EXPECT(g.shard_size(0) == 2 && g.shard_size(1) == 2 && g.shard_size(2) == 1);
  EXPECT(throws_invalid([] { Grid1xP::split(6, 5); }));
  std::vector<std::vector<double>> b = {{1}, {2}, {3}, {4}};
  EXPECT(tree_reduce(b, Precision::Double)[0] == 10.0);
  EXPECT(std::fabs(effective_bandwidth(128, 4096, 100, 4, 1.0) - 0.2114048) < 1e-12);
  auto u = uniform_fill(4, 7);
  EXPECT(u.size() == 4 && u[0] >= -1.0 && u[0] < 1.0);
  std::vector<ConfigResult> rows = {{parse_precision_config("ddddd"), 2.0, 2.0, 2.0, 0.0},
                                    {parse_precision_config("dssdd"), 1.0, 1.0, 1.0, 1e-8},
                                    {parse_precision_config("sssss"), 1.5, 1.5, 1.5, 1e-6}};
  auto front = pareto_front(rows);
  EXPECT(front.size() == 2);
  EXPECT(optimal_config(rows, 1e-7).render() == "dssdd");
  EXPECT(optimal_config(rows, 1e-9).render() == "ddddd");
  SweepReport rep = make_report(ProblemDims(3, 2, 4), MatvecKind::Forward, 1, 1e-7, rows);
  auto back = parse_sweep_csv(to_csv(rep));
  EXPECT(back.size() == 3 && back[1].config.render() == "dssdd" && back[2].rel_error == 1e-6);
  BlockVector v = BlockVector::time_double(2, 3, {1, 2, 3, 4, 5, 6});
  auto t = reorder(v, Layout::TOSI);
  EXPECT(t.f64[1] == 4 && reorder(t, Layout::SOTI).f64 == v.f64);
}

// direct block-Toeplitz products (dense_ref.hpp semantics), for the check only
static std::vector<double> dense(const BlockColumn& c, const std::vector<double>& x, bool fwd) {
  const auto& d = c.dims;
  std::vector<double> y((fwd ? d.n_d : d.n_m) * d.n_t, 0.0);
  for (std::size_t i = 0; i < d.n_t; ++i)
    for (std::size_t j = 0; j <= i; ++j)
      for (std::size_t col = 0; col < d.n_m; ++col)
        for (std::size_t r = 0; r < d.n_d; ++r) {
          if (fwd)
            y[r * d.n_t + i] += c.at(i - j, r, col) * x[col * d.n_t + j];
          else
            y[col * d.n_t + j] += c.at(i - j, r, col) * x[r * d.n_t + i];
        }
  return y;
}

static void gpu_checks() {
  const ProblemDims dims(16, 4, 32);
  BlockColumn col(dims, uniform_fill(dims.n_t * dims.n_d * dims.n_m, seed_stream(20250814, 0)));
  const auto m = uniform_fill(dims.n_m * dims.n_t, seed_stream(20250814, 1));
  const auto d = uniform_fill(dims.n_d * dims.n_t, seed_stream(20250814, 2));
  SpectralOperator op = setup_operator(col);
  EXPECT(op.bins_double.size() == dims.n_bins() * dims.n_d * dims.n_m);
  reset_cast_counter();
  auto F = forward_matvec(op, BlockVector::time_double(dims.n_m, dims.n_t, m), PrecisionConfig::all_double());
  auto A = adjoint_matvec(op, BlockVector::time_double(dims.n_d, dims.n_t, d), parse_precision_config("ddddd"));
  EXPECT(casts_performed() == 0);
  const double ef = relative_error(F.output.f64, dense(col, m, true));
  const double ea = relative_error(A.output.f64, dense(col, d, false));
  std::printf("  forward vs dense %.3e, adjoint vs dense %.3e\n", ef, ea);
  EXPECT(ef <= 1e-12 && ea <= 1e-12);
  double lhs = 0, rhs = 0;
  for (std::size_t i = 0; i < d.size(); ++i) lhs += F.output.f64[i] * d[i];
  for (std::size_t i = 0; i < m.size(); ++i) rhs += m[i] * A.output.f64[i];
  EXPECT(std::fabs(lhs - rhs) <= 1e-11 * std::fabs(lhs));
  // delta column: d_i = B m_i
  BlockColumn delta = BlockColumn::zeros(dims);
  for (std::size_t k = 0; k < dims.n_d * dims.n_m; ++k) delta.data[k] = col.data[k];
  auto Fd = forward_matvec(setup_operator(delta), BlockVector::time_double(dims.n_m, dims.n_t, m),
                           PrecisionConfig::all_double());
  EXPECT(relative_error(Fd.output.f64, dense(delta, m, true)) <= 1e-12);
  // partitions: p=1 bitwise, p=2,4 within 1e-12
  for (std::size_t p : {1u, 2u, 4u}) {
    auto pop = setup_partitioned(col, Grid1xP::split(p, dims.n_m));
    auto pf = forward_matvec_partitioned(pop, BlockVector::time_double(dims.n_m, dims.n_t, m), PrecisionConfig{});
    auto pa = adjoint_matvec_partitioned(pop, BlockVector::time_double(dims.n_d, dims.n_t, d), PrecisionConfig{});
    if (p == 1) EXPECT(pf.output.f64 == F.output.f64 && pa.output.f64 == A.output.f64);
    EXPECT(relative_error(pf.output.f64, F.output.f64) <= 1e-12);
    EXPECT(relative_error(pa.output.f64, A.output.f64) <= 1e-12);
  }
  // block (multi-RHS) matvecs: every RHS equals the single-RHS result to rounding
  {
    std::vector<BlockVector> ms, ds;
    for (int r = 0; r < 3; ++r) {
      ms.push_back(BlockVector::time_double(dims.n_m, dims.n_t, uniform_fill(dims.n_m * dims.n_t, 40 + r)));
      ds.push_back(BlockVector::time_double(dims.n_d, dims.n_t, uniform_fill(dims.n_d * dims.n_t, 50 + r)));
    }
    auto BF = forward_matvec_block(op, ms);
    auto BA = adjoint_matvec_block(op, ds);
    EXPECT(BF.size() == 3 && BA.size() == 3);
    for (int r = 0; r < 3; ++r) {
      EXPECT(relative_error(BF[r].f64, forward_matvec(op, ms[r], PrecisionConfig{}).output.f64) <= 1e-14);
      EXPECT(relative_error(BA[r].f64, adjoint_matvec(op, ds[r], PrecisionConfig{}).output.f64) <= 1e-14);
    }
  }
  // 2-D grid at 1 x 1 through NCCL (a real 1-rank communicator): equals the serial matvec bitwise
  {
    auto g = GridPxQ::split(2, 3, dims.n_d, dims.n_m);
    auto shards = shard_operator_2d(col, g);
    EXPECT(shards.size() == 6 && shards[4].dims.n_d == 2 && shards[4].dims.n_m == 5 && g.coords(4).second == 1);
    EXPECT(shards[4].at(3, 1, 2) == col.at(3, g.row_ranges[1].first + 1, g.col_ranges[1].first + 2));
    NcclGrid2D grid(1, 1, 0, NcclPartition::unique_id());
    const auto gf = grid.forward(op, m, PrecisionConfig{});
    const auto ga = grid.adjoint(op, d, PrecisionConfig{});
    EXPECT(gf == F.output.f64 && ga == A.output.f64);
  }
  // large results (>= 4 MB: F* at n_m*n_t = 600k) take the pinned-buffer + helper-thread path of
  // run_pipeline; they must equal the C ABI's own host-I/O result bitwise, repeatedly (the helper's
  // reused arena), and for F and F* with mixed configs too
  {
    const ProblemDims big(1000, 3, 600);
    BlockColumn bcol(big, uniform_fill(big.n_t * big.n_d * big.n_m, seed_stream(7, 0)));
    SpectralOperator bop = setup_operator(bcol, HostBins::Skip);
    const auto bm = uniform_fill(big.n_m * big.n_t, seed_stream(7, 1));
    const auto bd = uniform_fill(big.n_d * big.n_t, seed_stream(7, 2));
    for (const char* c : {"ddddd", "dssdd"}) {
      std::vector<double> want_a(big.n_m * big.n_t), want_f(big.n_d * big.n_t);
      detail::check(fmv_matvec(detail::thread_ctx(0), bop.handle(), FMV_ADJOINT, c, bd.data(), want_a.data(), 0,
                               nullptr));
      detail::check(fmv_matvec(detail::thread_ctx(0), bop.handle(), FMV_FORWARD, c, bm.data(), want_f.data(), 0,
                               nullptr));
      for (int rep = 0; rep < 3; ++rep) {
        auto ba = adjoint_matvec(bop, BlockVector::time_double(big.n_d, big.n_t, bd), parse_precision_config(c));
        auto bf = forward_matvec(bop, BlockVector::time_double(big.n_m, big.n_t, bm), parse_precision_config(c));
        EXPECT(ba.output.f64 == want_a);
        EXPECT(bf.output.f64 == want_f);
        EXPECT(ba.timings.total_s > 0);
      }
    }
  }
  // FFT facade round trip
  FftPlan fwd(16, 3, Precision::Double, FftDirection::Forward), inv(16, 3, Precision::Double, FftDirection::Inverse);
  auto x = uniform_fill(48, 3);
  auto X = forward_real_batched(fwd, x);
  auto xr = inverse_real_batched(inv, X);
  EXPECT(relative_error(xr, x) <= 1e-12);
  // GEMV facade: ConjTrans of [[i,0],[0,i]] times (1,1) = (-i,-i)
  std::vector<std::complex<double>> Am = {{0, 1}, {0, 0}, {0, 0}, {0, 1}}, xv = {{1, 0}, {1, 0}}, yv(2);
  gemv_batched_auto(GemvMode::ConjTrans, MatrixBatch<std::complex<double>>::tight(Am, 2, 2, 1),
                    VectorBatch<const std::complex<double>>::tight(xv, 2, 1),
                    VectorBatch<std::complex<double>>::tight(yv, 2, 1));
  EXPECT(yv[0] == std::complex<double>(0, -1) && yv[1] == std::complex<double>(0, -1));
  // sweep: 32 rows, baseline error 0, optimal within tolerance
  auto rows = sweep_configs(op, m, MatvecKind::Forward, 2, 1);
  EXPECT(rows.size() == 32 && rows[0].rel_error == 0.0);
  auto rep = make_report(dims, MatvecKind::Forward, 2, 1e-5, rows);
  EXPECT(std::find_if(rows.begin(), rows.end(), [&](auto& r) { return r.config == rep.chosen; })->rel_error <= 1e-5);
}

// FMV1 (include/fftmv/vector_io.hpp): round trips over every code, the named
// errors, and a file for the Python side to compare byte for byte.
static void fmv1_checks() {
  int n = 0;
  for (int lay = 0; lay < 2; ++lay)
    for (int prec = 0; prec < 2; ++prec)
      for (int dom = 0; dom < 2; ++dom) {
        BlockVector v;
        v.space_extent = 3 + lay;
        v.time_extent = 5 + prec;
        v.layout = lay ? Layout::TOSI : Layout::SOTI;
        v.precision = prec ? Precision::Single : Precision::Double;
        v.domain = dom ? Domain::Frequency : Domain::Time;
        auto x = uniform_fill(v.scalar_count(), 100 + n++);
        if (prec) v.f32.assign(x.begin(), x.end());
        else v.f64 = x;
        const BlockVector w = decode_vector(encode_vector(v));
        EXPECT(w.space_extent == v.space_extent && w.time_extent == v.time_extent && w.layout == v.layout &&
               w.precision == v.precision && w.domain == v.domain && w.f64 == v.f64 && w.f32 == v.f32);
      }
  auto throws = [](const std::string& s, const char* what) {
    try {
      (void)decode_vector(s);
    } catch (const std::invalid_argument& e) {
      return std::string(e.what()).find(what) != std::string::npos;
    }
    return false;
  };
  const std::string good = encode_vector(BlockVector::time_double(2, 3, uniform_fill(6, 7)));
  EXPECT(throws("", "bad magic") && throws("FMV2" + good.substr(4), "bad magic"));
  EXPECT(throws(good.substr(0, 20), "truncated file"));
  EXPECT(throws(good.substr(0, good.size() - 8), "truncated/oversized") && throws(good + "x", "truncated/oversized"));
  std::string bad = good;
  bad[4 + 16] = 2;
  EXPECT(throws(bad, "layout code out of range"));
  if (const char* path = std::getenv("FMV1_OUT")) {
    BlockVector v = BlockVector::time_double(4, 9, uniform_fill(36, 2025));
    save_vector(path, v);
    EXPECT(load_vector(path).f64 == v.f64);
  }
}

int main(int argc, char** argv) {
  host_checks();
  fmv1_checks();
  if (argc > 1 && std::strcmp(argv[1], "--gpu") == 0) gpu_checks();
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
