// test_engine_cpp.cpp — the reference's engine test cases
// (/root/reference/proj/tests/test_engine.cpp) re-hosted on the C++ host API
// (include/hpac/hpac.hpp) and run on the GPU. Each case cites the reference
// test it restates. Exit code = number of failed checks.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <vector>

#include "hpac/hpac.hpp"

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(cond)) {                                                          \
      ++g_fail;                                                             \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                       \
  } while (0)

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t count, const T* host = nullptr) : n(count) {
    cudaMalloc(&p, sizeof(T) * (n ? n : 1));
    if (host) cudaMemcpy(p, host, sizeof(T) * n, cudaMemcpyHostToDevice);
  }
  Dev(const std::vector<T>& v) : Dev(v.size(), v.data()) {}
  ~Dev() { cudaFree(p); }
  std::vector<T> get() const {
    std::vector<T> h(n);
    cudaMemcpy(h.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost);
    return h;
  }
};

using namespace hpac;

static GridConfig grid_of(int teams, int threads, int warp, int ipt) {
  GridConfig g;
  g.num_teams = teams;
  g.threads_per_team = threads;
  g.warp_size = warp;
  g.items_per_thread = ipt;
  return g;
}

// synthetic_reference (bench/synthetic.hpp:74-80), no contraction
static double synth_value(int prof, long long i, uint64_t seed) {
  if (prof == HPAC_SYNTH_CONSTANT) return 7.5;
  if (prof == HPAC_SYNTH_SLOW_DRIFT) {
    volatile double t = 1e-5 * (double)i;
    volatile double u = 1.0 + t;
    return 50.0 * u;
  }
  uint64_t x = seed ^ (uint64_t)i;
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  x ^= x >> 31;
  volatile double f = (double)(x >> 11) * 0x1.0p-53;
  return 1.0 + f;
}
static std::vector<double> synth_ref(int prof, uint64_t seed, long long n) {
  std::vector<double> o(n);
  for (long long i = 0; i < n; ++i) {
    volatile double t = 3.0 * synth_value(prof, i, seed);
    o[i] = t + 1.0;
  }
  return o;
}

static void baseline_accurate() {  // test_engine.cpp:63-72
  Dev<double> out(64);
  auto lr = run_region(grid_of(2, 8, 4, 4), 64, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_SLOW_DRIFT, 1, out.p), nullptr);
  CHECK(lr.stats.total_invocations == 64);
  CHECK(lr.stats.approx_invocations == 0);
  CHECK(out.get() == synth_ref(HPAC_SYNTH_SLOW_DRIFT, 1, 64));
}

static void taf_threshold_zero_noise() {  // :74-83
  Dev<double> out(128);
  auto spec = ApproxSpec::taf(3, 8, 0.0);
  auto lr = run_region(grid_of(2, 8, 4, 8), 128, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_NOISE, 99, out.p), &spec);
  CHECK(lr.stats.approx_invocations == 0);
  CHECK(out.get() == synth_ref(HPAC_SYNTH_NOISE, 99, 128));
}

static void taf_steady_state() {  // :85-100
  int h = 2, p = 3, cycles = 10;
  long long n = 8LL * cycles * (h + p);
  Dev<double> out(n);
  auto spec = ApproxSpec::taf(h, p, std::numeric_limits<double>::infinity());
  auto lr = run_region(grid_of(1, 8, 4, cycles * (h + p)), n, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_CONSTANT, 1, out.p), &spec);
  CHECK(lr.stats.total_invocations == (uint64_t)n);
  CHECK(lr.stats.approx_invocations == (uint64_t)(8LL * cycles * p));
  CHECK(out.get() == synth_ref(HPAC_SYNTH_CONSTANT, 1, n));
}

static void iact_constant_fixture() {  // :130-140
  Dev<double> out(64);
  auto spec = ApproxSpec::iact(2, 0.5);
  auto lr = run_region(grid_of(1, 4, 4, 16), 64, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_CONSTANT, 7, out.p), &spec);
  CHECK(lr.stats.approx_invocations == 60);
  CHECK(out.get() == synth_ref(HPAC_SYNTH_CONSTANT, 7, 64));
}

static void iact_shared_tables() {  // :142-178
  long long n = 16;
  std::vector<double> in(n), tab(n);
  for (long long i = 0; i < n; ++i) {
    long long step = i / 4, lane = i % 4;
    in[i] = (double)((step + lane) % 4);
    tab[i] = in[i] * 10.0;
  }
  Dev<double> din(in), dtab(tab), o1(n), o2(n);
  auto shared = ApproxSpec::iact(4, 0.0, 1);
  auto solo = ApproxSpec::iact(4, 0.0, 4);
  auto a = run_region(grid_of(1, 4, 4, 4), n, WorkMapping::kPerThread,
                      table_region(1, 1, din.p, dtab.p, o1.p), &shared);
  auto b = run_region(grid_of(1, 4, 4, 4), n, WorkMapping::kPerThread,
                      table_region(1, 1, din.p, dtab.p, o2.p), &solo);
  CHECK(a.stats.approx_invocations == 6);
  CHECK(b.stats.approx_invocations == 0);
  CHECK(o1.get() == o2.get());
}

static void iact_infinite_threshold() {  // :180-190
  Dev<double> out(128);
  auto spec = ApproxSpec::iact(2, std::numeric_limits<double>::infinity());
  auto lr = run_region(grid_of(1, 8, 8, 16), 128, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_NOISE, 13, out.p), &spec);
  CHECK(lr.stats.approx_invocations == 120);
}

static void perforation_untouched() {  // :192-208
  long long n = 32;
  std::vector<double> init(n, -1.0);
  Dev<double> out(init);
  auto spec = ApproxSpec::perfo(PerfoKind::kSmall, 4);
  auto lr = run_region(grid_of(1, 4, 4, 8), n, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_CONSTANT, 3, out.p), &spec);
  CHECK(lr.approx_rate() == 0.25);
  auto o = out.get();
  auto ref = synth_ref(HPAC_SYNTH_CONSTANT, 3, n);
  for (long long i = 0; i < n; ++i) CHECK((i / 4) % 4 == 3 ? o[i] == -1.0 : o[i] == ref[i]);
}

static void herded_vs_small_ragged() {  // :210-257
  long long n = 128;
  std::vector<int32_t> enc(n);
  std::vector<double> one(n, 1.0);
  for (long long i = 0; i < n; ++i) enc[i] = i % 2 == 0 ? 2 : 1;
  Dev<int32_t> denc(enc);
  Dev<double> tab(one), s1(std::vector<double>(n, 0.0)), s2(std::vector<double>(n, 0.0));
  auto small = ApproxSpec::perfo(PerfoKind::kSmall, 2);
  auto herded = ApproxSpec::perfo(PerfoKind::kHerdedSmall, 2);
  auto a = run_region(grid_of(1, 8, 8, 16), n, WorkMapping::kPerThread,
                      table_region(0, 1, nullptr, tab.p, s1.p, denc.p, HPAC_REGION_STORE_ACCUMULATE), &small);
  auto b = run_region(grid_of(1, 8, 8, 16), n, WorkMapping::kPerThread,
                      table_region(0, 1, nullptr, tab.p, s2.p, denc.p, HPAC_REGION_STORE_ACCUMULATE), &herded);
  CHECK(a.stats.divergent_warp_steps > 0);
  CHECK(b.stats.divergent_warp_steps == 0);
  std::mt19937_64 rng(505);
  for (int iter = 0; iter < 25; ++iter) {
    int teams = 1 + (int)(rng() % 3);
    int warp = 4 << (rng() % 2);
    int threads = warp * (1 + (int)(rng() % 2));
    long long m = 1 + (long long)(rng() % 300);
    int ipt = (int)((m + teams * threads - 1) / (teams * threads)) + (int)(rng() % 3) + 1;
    Dev<double> out(m);
    auto spec = ApproxSpec::perfo(rng() % 2 ? PerfoKind::kHerdedSmall : PerfoKind::kHerdedLarge,
                                  2 + (int)(rng() % 6));
    auto lr = run_region(grid_of(teams, threads, warp, ipt), m, WorkMapping::kPerThread,
                         synthetic_region(HPAC_SYNTH_NOISE, iter, out.p), &spec);
    CHECK(lr.stats.divergent_warp_steps == 0);
  }
}

static void warp_voting() {  // :259-298
  long long n = 256;
  std::vector<double> tab(n);
  for (long long i = 0; i < n; ++i) tab[i] = (i % 8) < 3 ? 1.0 + 0.37 * (double)i : 42.0;
  Dev<double> dtab(tab), ot(n), ow(n);
  auto ts = ApproxSpec::taf(2, 4, 0.05, Level::kThread);
  auto wsp = ApproxSpec::taf(2, 4, 0.05, Level::kWarp);
  auto t = run_region(grid_of(1, 8, 8, 32), n, WorkMapping::kPerThread, table_region(0, 1, nullptr, dtab.p, ot.p), &ts);
  auto w = run_region(grid_of(1, 8, 8, 32), n, WorkMapping::kPerThread, table_region(0, 1, nullptr, dtab.p, ow.p), &wsp);
  CHECK(t.stats.divergent_warp_steps > 0);
  CHECK(w.stats.divergent_warp_steps == 0);
  auto o = ow.get();
  bool forced = false;
  for (long long i = 0; i < n; ++i)
    if (i % 8 < 3 && o[i] != tab[i]) forced = true;
  CHECK(forced);
}

static void barrier_deadlock_model() {  // :300-328
  long long n = 32;
  std::vector<double> tab(n);
  for (long long i = 0; i < n; ++i) tab[i] = i % 2 == 0 ? 5.0 : 1.0 + 0.61 * (double)i;
  Dev<double> dtab(tab), o1(n), o2(n);
  auto ts = ApproxSpec::taf(2, 4, 0.01, Level::kThread);
  bool threw = false;
  try {
    run_region(grid_of(1, 2, 2, 16), n, WorkMapping::kPerThread,
               table_region(0, 1, nullptr, dtab.p, o1.p, nullptr, HPAC_REGION_BARRIER_IN_EVALUATE), &ts);
  } catch (const BarrierDivergenceError&) {
    threw = true;
  }
  CHECK(threw);
  auto team = ApproxSpec::taf(2, 4, 0.01, Level::kTeam);
  bool ok = true;
  try {
    run_region(grid_of(1, 2, 2, 16), n, WorkMapping::kPerThread,
               table_region(0, 1, nullptr, dtab.p, o2.p, nullptr, HPAC_REGION_BARRIER_IN_EVALUATE), &team);
  } catch (const SimtError&) {
    ok = false;
  }
  CHECK(ok);
}

static void team_vote_multiples() {  // :330-349
  long long n = 192;
  std::vector<double> tab(n);
  for (long long i = 0; i < n; ++i) tab[i] = (i % 8) < 5 ? 9.0 : 0.5 + 0.7 * (double)i;
  Dev<double> dtab(tab), o(n);
  auto spec = ApproxSpec::taf(1, 6, 0.01, Level::kTeam);
  auto lr = run_region(grid_of(1, 8, 4, 24), n, WorkMapping::kPerThread, table_region(0, 1, nullptr, dtab.p, o.p), &spec);
  CHECK(lr.stats.divergent_warp_steps == 0);
  CHECK(lr.stats.approx_invocations > 0);
  CHECK(lr.stats.approx_invocations % 8 == 0);
}

static void tail_masking() {  // :351-360
  Dev<double> out(9);
  auto spec = ApproxSpec::taf(1, 2, std::numeric_limits<double>::infinity(), Level::kWarp);
  auto lr = run_region(grid_of(1, 8, 8, 2), 9, WorkMapping::kPerThread,
                       synthetic_region(HPAC_SYNTH_CONSTANT, 2, out.p), &spec);
  CHECK(lr.stats.total_invocations == 9);
  CHECK(lr.stats.total_warp_steps == 2);
}

static void per_team_mapping() {  // :362-384
  long long n = 6;
  std::vector<double> tab(n);
  for (long long i = 0; i < n; ++i) tab[i] = (double)i;
  Dev<double> dtab(tab), o(n);
  auto lr = run_region(grid_of(2, 4, 4, 3), n, WorkMapping::kPerTeam, table_region(0, 1, nullptr, dtab.p, o.p), nullptr);
  CHECK(lr.stats.total_invocations == 24);
  CHECK(o.get() == tab);
}

static void arena_overflow() {  // :386-393
  GridConfig g = grid_of(1, 32, 32, 4);
  g.shared_mem_budget_bytes = 64;
  Dev<double> out(128);
  auto spec = ApproxSpec::taf(5, 4, 1.0);
  bool threw = false;
  try {
    run_region(g, 128, WorkMapping::kPerThread, synthetic_region(HPAC_SYNTH_CONSTANT, 1, out.p), &spec);
  } catch (const ArenaOverflowError& e) {
    threw = e.required_bytes == 112 && e.available_bytes == 64;
  }
  CHECK(threw);
}

static void deterministic() {  // :395-407
  auto once = [] {
    Dev<double> out(128);
    auto spec = ApproxSpec::taf(2, 4, 0.01);
    auto lr = run_region(grid_of(2, 8, 4, 8), 128, WorkMapping::kPerThread,
                         synthetic_region(HPAC_SYNTH_SLOW_DRIFT, 11, out.p), &spec);
    return std::make_pair(out.get(), lr.stats.approx_invocations);
  };
  CHECK(once() == once());
}

static void directives_and_grid() {
  auto s = parse_directive("memo(in:2:0.5f:4) level(warp) in(input[i*5:5:N]) out(output1[i])");
  CHECK(s.technique() == Technique::kIact && s.level() == Level::kWarp);
  CHECK(unparse(s) == "memo(in:2:0.5:4) level(warp) in(input[i*5:5:N]) out(output1[i])");
  bool threw = false;
  try {
    parse_directive("memo(out:1:2:3)");
  } catch (const DirectiveError& e) {
    threw = e.code == 12;
  }
  CHECK(threw);
  WorkMapping m;
  GridConfig g = resolve_grid("binomial", 1 << 20, nullptr, &m);
  CHECK(m == WorkMapping::kPerTeam && g.num_teams == (1 << 20) / 8);
}

static void kmeans_small() {  // test_bench.cpp:139-163
  std::vector<double> pts(512 * 2);
  hpac_make_blobs(512, 2, 4, 11, 14.0, pts.data());
  Dev<double> dp(pts), dc(8);
  Dev<int32_t> da(512);
  auto r = kmeans_benchmark(dp.p, 512, 2, 4, dc.p, da.p, grid_of(2, 64, 32, 4), nullptr);
  CHECK(r.converged && r.iterations <= 2);
}

static void lavamd_levels() {  // extension: TAF at warp vs team, staging outside the region
  const int b1 = 4, P = 64, nb = b1 * b1 * b1;
  std::vector<double> rv(nb * P * 4), qv(nb * P);
  hpac_make_lavamd(b1, P, 3, rv.data(), qv.data());
  const std::vector<double> zero(nb * P * 4, 0.0);
  Dev<double> drv(rv), dqv(qv), fe(zero), fw(zero), ft(zero);
  GridConfig g = grid_of(nb, P, 32, 1);
  auto e = run_region(g, nb, WorkMapping::kPerTeam, lavamd_region(drv.p, dqv.p, fe.p, b1, P), nullptr);
  ApproxSpec w = parse_directive("memo(out:2:4:0.2) out(fv[i:4]) level(warp)");
  ApproxSpec t = parse_directive("memo(out:2:4:0.2) out(fv[i:4]) level(team)");
  auto rw = run_region(g, nb, WorkMapping::kPerTeam, lavamd_region(drv.p, dqv.p, fw.p, b1, P), &w);
  auto rt = run_region(g, nb, WorkMapping::kPerTeam, lavamd_region(drv.p, dqv.p, ft.p, b1, P), &t);
  CHECK(e.stats.approx_invocations == 0 && e.stats.total_invocations == rw.stats.total_invocations);
  CHECK(rw.stats.divergent_warp_steps == 0 && rt.stats.divergent_warp_steps == 0);
  CHECK(rw.stats.approx_invocations % 32 == 0 && rt.stats.approx_invocations % P == 0);
  CHECK(rt.stats.approx_invocations > 0);
  bool threw = false;
  try {
    run_region(grid_of(nb, 2 * P, 32, 1), nb, WorkMapping::kPerTeam, lavamd_region(drv.p, dqv.p, fe.p, b1, P),
               nullptr);
  } catch (const ConfigError&) {
    threw = true;  // particles must equal threads_per_team
  }
  CHECK(threw);
}

static void host_team_ranges() {  // multi-GPU split with host buffers (hpac_run_region_host_teams)
  const long long n = 40 * 16 - 9;
  std::vector<double> opts(n * 5);
  hpac_make_binomial_portfolio(n, 5, 0.002, opts.data());
  GridConfig g = grid_of(40, 64, 32, 16);
  ApproxSpec s = parse_directive("memo(in:4:0.4) level(team) in(o[i:5]) out(p[i])");
  std::vector<double> whole(n, -1.0), parts(n, -1.0);
  auto rw = run_region_host(g, n, WorkMapping::kPerTeam, binomial_region(opts.data(), 64, whole.data()), &s);
  unsigned long long approx = 0, total = 0;
  for (int a = 0; a < 40; a += 13) {
    const int b = a + 13 < 40 ? a + 13 : 40;
    auto r = run_region_host_teams(g, n, WorkMapping::kPerTeam,
                                   binomial_region(opts.data(), 64, parts.data()), &s, a, b);
    approx += r.stats.approx_invocations;
    total += r.stats.total_invocations;
  }
  CHECK(parts == whole);
  CHECK(approx == rw.stats.approx_invocations && total == rw.stats.total_invocations);
}

int main() {
  std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"baseline_accurate", baseline_accurate}, {"taf_threshold_zero_noise", taf_threshold_zero_noise},
      {"taf_steady_state", taf_steady_state}, {"iact_constant_fixture", iact_constant_fixture},
      {"iact_shared_tables", iact_shared_tables}, {"iact_infinite_threshold", iact_infinite_threshold},
      {"perforation_untouched", perforation_untouched}, {"herded_vs_small_ragged", herded_vs_small_ragged},
      {"warp_voting", warp_voting}, {"barrier_deadlock_model", barrier_deadlock_model},
      {"team_vote_multiples", team_vote_multiples}, {"tail_masking", tail_masking},
      {"per_team_mapping", per_team_mapping}, {"arena_overflow", arena_overflow},
      {"deterministic", deterministic}, {"directives_and_grid", directives_and_grid},
      {"kmeans_small", kmeans_small}, {"lavamd_levels", lavamd_levels},
      {"host_team_ranges", host_team_ranges}};
  for (auto& [name, fn] : cases) {
    int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "FAIL %s: exception %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
  return g_fail;
}
