// Deterministic replay backend (see include/gpuos/replay.hpp).
//
// Reference behaviour reproduced here, by file:line of device.cpp:
//   slot capacity as an exact fraction ........................ :94-119
//   submit: validate, sort TPCs, priority-ordered residency .... :121-163
//   pause keeps in-flight blocks, starts none .................. :165-171
//   block start: prelude when atomized, latency at current f ... :173-186
//   refill from the first eligible resident atom, no bypass .... :188-206
//   completion callback fired synchronously from the event ..... :208-219
//   frequency switch with replace-pending semantics ............ :221-242
//   piecewise accounting clamped at the metrics horizon ........ :264-275
//   (t, seq) event order, one seq counter for atoms and events . :232-262
#include <algorithm>
#include <numeric>

#include "gpuos/replay.hpp"

namespace gpuos {

namespace {
// Heap order: the earliest (t, seq) on top.
inline bool later(const auto& a, const auto& b) {
  return a.t != b.t ? a.t > b.t : a.seq > b.seq;
}
}  // namespace

void DeviceEngine::Load::add_share(int o) {
  long n = num * o + den;
  long d = den * o;
  long g = std::gcd(n, d);
  num = n / g;
  den = d / g;
}

void DeviceEngine::Load::drop_share(int o) {
  long n = num * o - den;
  long d = den * o;
  if (n < 0) throw InvariantError("TPC slot accounting went negative");
  if (n == 0) {
    num = 0;
    den = 1;
    return;
  }
  long g = std::gcd(n, d);
  num = n / g;
  den = d / g;
}

DeviceEngine::DeviceEngine(DeviceTopology topo, FrequencyDomain freq,
                           PowerModel power)
    : topo_(topo), freq_(std::move(freq)), power_(power) {
  topo_.validate();
  freq_.validate();
  mhz_ = freq_.f_max();
  tpc_.resize(static_cast<std::size_t>(topo_.total_tpcs()));
}

KernelId DeviceEngine::register_kernel(const SimKernelSpec& spec) {
  spec.validate();
  kernels_.push_back(spec);
  executed_.push_back(0);
  return static_cast<KernelId>(kernels_.size() - 1);
}

long DeviceEngine::blocks_executed(KernelId k) const { return executed_.at(k); }

void DeviceEngine::push(SimTime t, Kind kind, int tpc, std::uint32_t ref) {
  heap_.push_back(Event{t, seq_++, kind, tpc, ref});
  std::push_heap(heap_.begin(), heap_.end(),
                 [](const Event& a, const Event& b) { return later(a, b); });
}

AtomId DeviceEngine::submit_atom(KernelId kernel, long lo, long hi,
                                 const std::vector<int>& tpcs, int priority,
                                 bool atomized, std::uint64_t tag) {
  const SimKernelSpec& spec = kernels_.at(kernel);
  if (tpcs.empty()) throw ConfigError("atom needs a non-empty TPC set");
  if (lo < 0 || hi <= lo || hi > spec.total_blocks)
    throw ConfigError("atom block range out of bounds");
  const int ntpc = topo_.total_tpcs();
  for (int t : tpcs)
    if (t < 0 || t >= ntpc) throw ConfigError("TPC id out of range");

  const AtomId id = static_cast<AtomId>(atoms_.size());
  {
    Atom a;
    a.kernel = kernel;
    a.cursor = lo;
    a.end = hi;
    a.tpcs = tpcs;
    std::sort(a.tpcs.begin(), a.tpcs.end());
    a.priority = priority;
    a.seq = seq_++;
    a.tag = tag;
    a.dispatched = clock_;
    a.atomized = atomized;
    a.held = held_next_;
    atoms_.push_back(std::move(a));
  }
  const Atom& me = atoms_[id];
  // Residency order (priority desc, seq asc). Every resident atom is older
  // than this one, so it goes after all atoms of equal or higher priority.
  for (int t : me.tpcs) {
    auto& q = tpc_[t].queue;
    auto pos = std::find_if(q.begin(), q.end(), [&](AtomId other) {
      const Atom& o = atoms_[other];
      return o.priority < me.priority ||
             (o.priority == me.priority && o.seq > me.seq);
    });
    q.insert(pos, id);
  }
  for (int t : me.tpcs) refill(t);  // refill never appends to atoms_
  if (atoms_[id].cursor == atoms_[id].end && atoms_[id].running == 0)
    throw InvariantError("atom completed at submit");
  return id;
}

AtomId DeviceEngine::submit_chained(AtomId after, KernelId kernel, long lo, long hi,
                                    const std::vector<int>& tpcs, int priority,
                                    bool atomized, std::uint64_t tag, bool /*chain_head*/,
                                    bool /*no_early*/) {
  if (after == kNoAtom || atoms_.at(after).finished)
    return submit_atom(kernel, lo, hi, tpcs, priority, atomized, tag);
  if (atoms_[after].succ != kNoAtom) throw InvariantError("atom already has a successor");
  // Resident but held: refill() skips it until the predecessor retires.
  const AtomId id = static_cast<AtomId>(atoms_.size());
  atoms_[after].succ = id;
  held_next_ = true;
  const AtomId got = submit_atom(kernel, lo, hi, tpcs, priority, atomized, tag);
  held_next_ = false;
  if (got != id) throw InvariantError("chained atom id mismatch");
  return id;
}

void DeviceEngine::set_atom_paused(AtomId atom, bool paused) {
  Atom& a = atoms_.at(atom);
  if (a.finished || a.paused == paused) return;
  a.paused = paused;
  if (paused) return;
  const std::vector<int> order = a.tpcs;
  for (int t : order) refill(t);
}

void DeviceEngine::launch_block(int tpc, AtomId id) {
  TpcState& ts = tpc_[tpc];
  Atom& a = atoms_[id];
  const SimKernelSpec& spec = kernels_[a.kernel];
  account_to(clock_);
  ts.load.add_share(spec.occupancy_per_tpc);
  if (ts.running++ == 0) ++busy_tpcs_;
  ++a.running;
  ++a.cursor;
  ++executed_[a.kernel];
  Duration d = block_latency(spec, mhz_, freq_);
  if (a.atomized) d += spec.prelude_overhead;
  push(clock_ + d, Kind::BlockDone, tpc, id);
}

void DeviceEngine::refill(int tpc) {
  TpcState& ts = tpc_[tpc];
  for (;;) {
    const Atom* pick = nullptr;
    AtomId pick_id = 0;
    for (AtomId id : ts.queue) {
      const Atom& a = atoms_[id];
      if (!a.paused && !a.held && a.cursor < a.end) {
        pick = &a;
        pick_id = id;
        break;
      }
    }
    // No lower-priority atom may bypass the chosen one, fit or not.
    if (pick == nullptr) return;
    if (!ts.load.admits(kernels_[pick->kernel].occupancy_per_tpc)) return;
    launch_block(tpc, pick_id);
  }
}

void DeviceEngine::retire(AtomId id) {
  Atom& a = atoms_[id];
  a.finished = true;
  for (int t : a.tpcs) {
    auto& q = tpc_[t].queue;
    q.erase(std::remove(q.begin(), q.end(), id), q.end());
  }
  if (a.succ != kNoAtom) {  // its chained successor starts now
    Atom& s = atoms_[a.succ];
    s.held = false;
    const std::vector<int> order = s.tpcs;
    for (int t : order) refill(t);
  }
  if (on_complete_) {
    const AtomCompletion c{id, atoms_[id].tag, atoms_[id].dispatched, clock_};
    on_complete_(c);
  }
}

SimTime DeviceEngine::request_frequency(FreqMhz f) {
  if (!freq_.supports(f)) throw ConfigError("unsupported frequency");
  if (f == mhz_) {
    pending_.reset();
    ++switch_gen_;
    return clock_;
  }
  if (pending_ && pending_->first == f) return pending_->second;
  const SimTime effective = clock_ + freq_.switch_latency;
  pending_ = std::make_pair(f, effective);
  push(effective, Kind::Clock, 0, ++switch_gen_);
  return effective;
}

void DeviceEngine::schedule_call(SimTime t, std::function<void()> fn) {
  if (t < clock_) throw InvariantError("scheduling a call in the past");
  std::uint32_t slot;
  if (!free_calls_.empty()) {
    slot = free_calls_.back();
    free_calls_.pop_back();
    calls_[slot] = std::move(fn);
  } else {
    slot = static_cast<std::uint32_t>(calls_.size());
    calls_.push_back(std::move(fn));
  }
  push(t, Kind::Call, 0, slot);
}

void DeviceEngine::account_to(SimTime t) {
  SimTime upto = t;
  if (horizon_ >= 0 && horizon_ < upto) upto = horizon_;
  if (upto > accounted_) {
    const Duration dt = upto - accounted_;
    const double dt_s = static_cast<double>(dt) / 1e9;
    joules_ += power_.watts(busy_tpcs_, mhz_, freq_.f_max()) * dt_s;
    busy_tpc_ns_ += static_cast<double>(busy_tpcs_) * dt;
    residency_[mhz_] += dt;
  }
  if (t > accounted_) accounted_ = t;
}

bool DeviceEngine::step() {
  if (heap_.empty()) return false;
  std::pop_heap(heap_.begin(), heap_.end(),
                [](const Event& a, const Event& b) { return later(a, b); });
  const Event e = heap_.back();
  heap_.pop_back();
  account_to(e.t);
  clock_ = e.t;
  switch (e.kind) {
    case Kind::BlockDone: {
      const AtomId id = e.ref;
      TpcState& ts = tpc_[e.tpc];
      ts.load.drop_share(kernels_[atoms_[id].kernel].occupancy_per_tpc);
      if (--ts.running == 0) --busy_tpcs_;
      --atoms_[id].running;
      refill(e.tpc);
      const Atom& a = atoms_[id];
      if (a.running == 0 && a.cursor == a.end && !a.finished) retire(id);
      break;
    }
    case Kind::Clock:
      if (e.ref == switch_gen_ && pending_) {
        mhz_ = pending_->first;
        pending_.reset();
      }
      break;
    case Kind::Call: {
      std::function<void()> fn = std::move(calls_[e.ref]);
      calls_[e.ref] = nullptr;
      free_calls_.push_back(e.ref);
      fn();
      break;
    }
  }
  return true;
}

void DeviceEngine::run_all() {
  while (step()) {
  }
}

}  // namespace gpuos
