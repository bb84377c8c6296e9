// ttkv_sim.cpp -- the reference's two-lane timing model for the C++ drop-in.
//
// Restates sim.cpp:16-196 (simulate_serial / simulate_pipelined,
// aggregate_run, dump_timeline) so harness code written against the
// reference's sim.hpp links against libttkv.so.  Same arithmetic in the same
// order as the reference, so modeled timelines agree bit for bit; on B200 the
// harness reports measured step latencies next to them
// (paper_2604_19769_b200/harness.py).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <numeric>
#include <ostream>
#include <unordered_map>

#include "ttkv/gpu_dropin.hpp"

namespace ttkv {
namespace {

void require_rates(const LinkModel& link, double rate) {
  if (link.bandwidth <= 0 || rate <= 0)
    throw ConfigError("simulate: bandwidth and compute_rate must be positive");
  if (link.fixed_latency < 0) throw ConfigError("simulate: fixed_latency must be non-negative");
}

void require_matched_labels(const StepWorkload& w) {
  for (const WorkItem& t : w.transfer_items) {
    bool found = false;
    for (const WorkItem& c : w.compute_items) found = found || c.label == t.label;
    if (!found)
      throw Error("workload: transfer item '" + t.label + "' has no matching compute item");
  }
}

// Both schedules: the transfer lane streams every transfer item back to back;
// the compute lane starts after all transfers (serial) or, per item, once the
// lane is free and its own transfer has landed (pipelined).
PipelineTimeline run_lanes(const StepWorkload& w, const LinkModel& link, double rate,
                           bool overlap) {
  require_rates(link, rate);
  require_matched_labels(w);
  PipelineTimeline tl;
  std::unordered_map<std::string, double> landed;
  double t = 0.0;
  for (const WorkItem& item : w.transfer_items) {
    const double dur = link.fixed_latency + item.amount / link.bandwidth;
    tl.events.push_back({TimelineEvent::Lane::Transfer, item.label, t, t + dur});
    t += dur;
    landed[item.label] = t;
  }
  tl.total_transfer = t;

  std::vector<double> begin(w.compute_items.size());
  double lane = overlap ? 0.0 : tl.total_transfer;
  for (std::size_t i = 0; i < w.compute_items.size(); ++i) {
    const WorkItem& item = w.compute_items[i];
    double start = lane;
    if (overlap) {
      const auto it = landed.find(item.label);
      if (it != landed.end()) start = std::max(start, it->second);
    }
    const double dur = item.amount / rate;
    tl.events.push_back({TimelineEvent::Lane::Compute, item.label, start, start + dur});
    begin[i] = start;
    lane = start + dur;
    tl.total_compute += dur;
  }
  tl.total_latency = overlap ? std::max(lane, tl.total_transfer) : lane;

  // stall of each fetched block against the zero-transfer schedule
  double ideal = 0.0, stall = 0.0;
  std::size_t fetched = 0;
  for (std::size_t i = 0; i < w.compute_items.size(); ++i) {
    if (landed.count(w.compute_items[i].label)) {
      stall += begin[i] - ideal;
      ++fetched;
    }
    ideal += w.compute_items[i].amount / rate;
  }
  tl.mean_transfer_stall = fetched ? stall / fetched : 0.0;
  tl.idle_fraction =
      tl.total_latency > 0 ? (tl.total_latency - tl.total_compute) / tl.total_latency : 0.0;
  return tl;
}

}  // namespace

PipelineTimeline simulate_serial(const StepWorkload& workload, const LinkModel& link,
                                 double compute_rate) {
  return run_lanes(workload, link, compute_rate, false);
}

PipelineTimeline simulate_pipelined(const StepWorkload& workload, const LinkModel& link,
                                    double compute_rate) {
  return run_lanes(workload, link, compute_rate, true);
}

double TrafficLedger::total_bytes() const {
  return std::accumulate(step_bytes.begin(), step_bytes.end(), 0.0);
}

double TrafficLedger::total_baseline_bytes() const {
  return std::accumulate(baseline_step_bytes.begin(), baseline_step_bytes.end(), 0.0);
}

RunSummary aggregate_run(const std::vector<PipelineTimeline>& timelines,
                         const TrafficLedger& ledger) {
  if (timelines.empty()) throw Error("aggregate_run: no timelines");
  const std::size_t warm = timelines.size() >= 25 ? 5 : 0;  // warm-up steps dropped
  std::vector<double> lat;
  for (std::size_t i = warm; i < timelines.size(); ++i) lat.push_back(timelines[i].total_latency);
  std::vector<double> order = lat;
  std::sort(order.begin(), order.end());
  const auto rank = static_cast<std::size_t>(std::ceil(0.95 * static_cast<double>(order.size())));
  RunSummary s;
  s.steps = timelines.size();
  s.p95_latency = order[rank == 0 ? 0 : rank - 1];  // nearest rank
  const double sum = std::accumulate(lat.begin(), lat.end(), 0.0);
  s.mean_latency = sum / static_cast<double>(lat.size());
  s.tokens_per_second = sum > 0 ? static_cast<double>(lat.size()) / sum : 0.0;
  s.total_h2g_bytes = ledger.total_bytes();
  const double base = ledger.total_baseline_bytes();
  s.traffic_reduction_vs_baseline =
      s.total_h2g_bytes > 0 ? base / s.total_h2g_bytes
                            : (base > 0 ? std::numeric_limits<double>::infinity() : 1.0);
  return s;
}

void dump_timeline(std::ostream& os, const PipelineTimeline& timeline) {
  char a[64], b[64];
  for (const TimelineEvent& e : timeline.events) {
    std::snprintf(a, sizeof(a), "%.9e", e.start);
    std::snprintf(b, sizeof(b), "%.9e", e.finish);
    os << (e.lane == TimelineEvent::Lane::Transfer ? "transfer" : "compute") << '\t' << e.label
       << '\t' << a << '\t' << b << '\n';
  }
}

}  // namespace ttkv
