// ledger.cpp — the IterationRecord ledger on the host:
// format_csv (runner.cpp:55-80) and summarize (runner.cpp:89-113) with the
// reference's byte format, so device runs can be diffed against `sparsim run`
// output. Doubles use std::to_chars' shortest round-trip form, as the
// reference's format_double (runner.cpp:27-31).
#include <charconv>
#include <cstring>
#include <string>

#include "exdyna.h"

namespace {

std::string fmt_double(double v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

}  // namespace

extern "C" {

int exd_format_csv(const exd_record* recs, int64_t count, char* out, size_t cap, size_t* len) {
  if (count < 0 || (count > 0 && !recs)) return EXD_EINVAL;
  std::string csv = "t,k_prime,density,eps,m_t,C_t,f_t,global_err,delta,loss\n";
  for (int64_t i = 0; i < count; ++i) {
    const exd_record& r = recs[i];
    csv += std::to_string(r.t);
    csv += ',';
    csv += std::to_string(r.k_prime);
    csv += ',';
    csv += fmt_double(r.density);
    csv += ',';
    csv += fmt_double(r.eps);
    csv += ',';
    csv += std::to_string(r.m_t);
    csv += ',';
    csv += std::to_string(r.c_t);
    csv += ',';
    csv += fmt_double(r.f_t);
    csv += ',';
    csv += fmt_double(r.global_err);
    csv += ',';
    csv += fmt_double(r.delta);
    csv += ',';
    if (r.has_loss) csv += fmt_double(r.loss);
    csv += '\n';
  }
  if (len) *len = csv.size();
  if (out && cap) {
    const size_t n = csv.size() < cap - 1 ? csv.size() : cap - 1;
    std::memcpy(out, csv.data(), n);
    out[n] = 0;
  }
  return EXD_OK;
}

int exd_summarize(const exd_record* recs, int64_t count, exd_run_stats* s) {
  if (!s || count < 0 || (count > 0 && !recs)) return EXD_EINVAL;
  std::memset(s, 0, sizeof(*s));
  s->iterations = count;
  if (count == 0) return EXD_OK;
  double idle = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const exd_record& r = recs[i];
    s->mean_density += r.density;
    s->mean_f += r.f_t;
    s->mean_eps += r.eps;
    s->duplicates += r.duplicates;
    s->adjust_moves += r.adjust_moves;
    s->adjust_skips += r.adjust_skips;
    s->cap_hits += r.cap_hits;
    idle += r.idle_workers;
  }
  const double n = (double)count;
  s->mean_density /= n;
  s->mean_f /= n;
  s->mean_eps /= n;
  s->mean_idle_workers = idle / n;
  s->final_delta = recs[count - 1].delta;
  s->final_global_err = recs[count - 1].global_err;
  s->has_final_loss = recs[count - 1].has_loss;
  s->final_loss = recs[count - 1].loss;
  return EXD_OK;
}

}  // extern "C"
