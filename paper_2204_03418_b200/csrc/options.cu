// options.cu — the library's documented planner / launch options (include/co.h
// co_set_option).  The release library reads no environment variable: these
// named switches, set through the C ABI, are its only knobs.  Each one selects
// among the sm_100a kernels or launch modes; none skips work or changes a
// result beyond the fp32 summation order.
//
// Builds with -DCO_EXPERIMENTS (build.py --variant exp --define CO_EXPERIMENTS)
// additionally read the A/B experiment variables through CO_EXP() (common.cuh);
// the release build compiles those reads out.
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "co.h"

namespace co {

namespace {

struct OptDef {
  const char* name;
  int64_t dflt, lo, hi;
};

// order == enum Opt (common.cuh)
constexpr OptDef kOpts[OPT_COUNT] = {
    {"tc_mode", 0, 0, 1},     {"khalo", 1, 0, 1},       {"pair", 0, 0, 2},       {"kpair", 0, 0, 2},
    {"eg", 0, 0, 4},          {"mc", 1, 1, 8},          {"pdl", 1, 0, 1},        {"chunk", 1, 0, 1},
    {"chunk_flat", 0, 0, 1},  {"chunk_st", 0, 0, 1},    {"chunk_t", 0, 0, 1 << 20},
    {"pool_band", 1, 0, 1},   {"pool_vh", -1, -1, 1},   {"pool_g", 0, 0, 32},    {"log", 0, 0, 1},
    {"stem", 1, 0, 1},        {"dw_seg", 1, 0, 1},
    {"mha_ring", 1, 0, 1},    {"pool_seg", 1, 0, 1},
};

std::atomic<int64_t> g_val[OPT_COUNT] = {};
std::atomic<bool> g_init{false};

void init_once() {
  bool expect = false;
  if (g_init.compare_exchange_strong(expect, true))
    for (int i = 0; i < OPT_COUNT; ++i) g_val[i].store(kOpts[i].dflt);
}

int find(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < OPT_COUNT; ++i)
    if (!std::strcmp(kOpts[i].name, name)) return i;
  return -1;
}

}  // namespace

// graph capture on this thread without programmatic dependent launch (the
// fallback when a driver cannot instantiate captured PDL edges)
thread_local int t_no_pdl = 0;
void set_thread_no_pdl(int v) { t_no_pdl = v; }

int64_t option(Opt o) {
  init_once();
  if (o == OPT_PDL && t_no_pdl) return 0;
  return g_val[o].load(std::memory_order_relaxed);
}

#ifdef CO_EXPERIMENTS
int experiment_knob(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
#endif

}  // namespace co

int co_set_option_impl(const char* name, int64_t value, std::string& err) {
  if (!name) {                                       // NULL: every option back to its default
    co::init_once();
    for (int i = 0; i < co::OPT_COUNT; ++i) co::g_val[i].store(co::kOpts[i].dflt);
    return CO_OK;
  }
  const int i = co::find(name);
  if (i < 0) { err = std::string("unknown option ") + (name ? name : "(null)"); return CO_ERR_ARG; }
  if (value < co::kOpts[i].lo || value > co::kOpts[i].hi) {
    err = std::string("option ") + name + " out of range";
    return CO_ERR_ARG;
  }
  co::init_once();
  co::g_val[i].store(value);
  return CO_OK;
}

int co_get_option_impl(const char* name, int64_t* value, std::string& err) {
  const int i = co::find(name);
  if (i < 0 || !value) { err = std::string("unknown option ") + (name ? name : "(null)"); return CO_ERR_ARG; }
  *value = co::option(co::Opt(i));
  return CO_OK;
}

int co_option_count_impl() { return co::OPT_COUNT; }
const char* co_option_name_impl(int i) { return (i >= 0 && i < co::OPT_COUNT) ? co::kOpts[i].name : nullptr; }
