// Compiled engine of the pipeline simulator (host code): the non-preemptive list scheduler that
// kvoverlap.pipesim runs as `_engine.pyx` beside its pure-Python `_engine_py.py` (engine.py:45-76),
// restated in C++ with the same results bit for bit (tests/test_pipesim_cpu.py, and the reference's own
// engine-parity tests through tests/refshim).
//
// Semantics (_engine_py.py:18-90): whenever a resource is idle it starts the ready task with the smallest
// (priority, id); every resource finishing at the same instant completes before the next dispatch, so
// simultaneous completions see one consistent ready set.  Times are doubles (start = now, end = now +
// duration), compared exactly, as in Python.

#include <functional>
#include <queue>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kvpr_internal.h"

extern "C" {

int kvpr_list_schedule(long long n, const long long* resource, const double* duration, const long long* priority,
                       const long long* dep_indptr, const long long* dep_indices, int n_resources, double* start,
                       double* end) {
  kvpr::clear_error();
  if (n < 0 || n_resources <= 0 || (n > 0 && (resource == nullptr || duration == nullptr || priority == nullptr ||
                                              dep_indptr == nullptr || start == nullptr || end == nullptr))) {
    kvpr::set_error("list_schedule: bad arguments (n=%lld, n_resources=%d)", n, n_resources);
    return KVPR_EINVAL;
  }
  if (n == 0) return KVPR_OK;
  // children of every task as CSR (two passes, no per-task allocation)
  std::vector<long long> indeg(n), child_ptr(n + 1, 0);
  for (long long i = 0; i < n; ++i) {
    if (resource[i] < 0 || resource[i] >= n_resources || dep_indptr[i + 1] < dep_indptr[i]) {
      kvpr::set_error("list_schedule: task %lld has resource %lld or a bad dependency range", i, resource[i]);
      return KVPR_EINVAL;
    }
    indeg[i] = dep_indptr[i + 1] - dep_indptr[i];
    for (long long p = dep_indptr[i]; p < dep_indptr[i + 1]; ++p) {
      const long long d = dep_indices[p];
      if (d < 0 || d >= n) {
        kvpr::set_error("list_schedule: task %lld depends on %lld (out of range)", i, d);
        return KVPR_EINVAL;
      }
      ++child_ptr[d + 1];
    }
  }
  for (long long i = 0; i < n; ++i) child_ptr[i + 1] += child_ptr[i];
  std::vector<long long> child(child_ptr[n]), fill(child_ptr.begin(), child_ptr.end() - 1);
  for (long long i = 0; i < n; ++i)
    for (long long p = dep_indptr[i]; p < dep_indptr[i + 1]; ++p) child[fill[dep_indices[p]]++] = i;
  // ready queues ordered by (priority, id): one packed int64 key priority * n + id when the priorities
  // fit (as the reference's compiled engine does), else (priority, id) pairs -- the same order
  long long pmin = priority[0], pmax = priority[0];
  for (long long i = 1; i < n; ++i) {
    pmin = priority[i] < pmin ? priority[i] : pmin;
    pmax = priority[i] > pmax ? priority[i] : pmax;
  }
  const bool packed = pmin >= 0 && pmax <= (1LL << 62) / n;
  std::vector<double> running_end(n_resources, 0.0);
  std::vector<long long> running_id(n_resources, -1);
  long long completed = 0;
  auto run = [&](auto& ready, auto key, auto id_of) {
    for (long long i = 0; i < n; ++i)
      if (indeg[i] == 0) ready[resource[i]].push(key(i));
    auto dispatch = [&](double now) {
      for (int r = 0; r < n_resources; ++r) {
        if (running_id[r] < 0 && !ready[r].empty()) {
          const long long i = id_of(ready[r].top());
          ready[r].pop();
          start[i] = now;
          end[i] = now + duration[i];
          running_id[r] = i;
          running_end[r] = end[i];
        }
      }
    };
    dispatch(0.0);
    for (;;) {
      bool any = false;
      double t = 0.0;
      for (int r = 0; r < n_resources; ++r)
        if (running_id[r] >= 0 && (!any || running_end[r] < t)) {
          t = running_end[r];
          any = true;
        }
      if (!any) break;
      for (int r = 0; r < n_resources; ++r) {
        if (running_id[r] >= 0 && running_end[r] == t) {
          const long long i = running_id[r];
          running_id[r] = -1;
          ++completed;
          for (long long p = child_ptr[i]; p < child_ptr[i + 1]; ++p)
            if (--indeg[child[p]] == 0) ready[resource[child[p]]].push(key(child[p]));
        }
      }
      dispatch(t);
    }
  };
  if (packed) {
    std::vector<std::priority_queue<long long, std::vector<long long>, std::greater<long long>>> ready(n_resources);
    run(ready, [&](long long i) { return priority[i] * n + i; }, [&](long long k) { return k % n; });
  } else {
    using Key = std::pair<long long, long long>;
    std::vector<std::priority_queue<Key, std::vector<Key>, std::greater<Key>>> ready(n_resources);
    run(ready, [&](long long i) { return Key(priority[i], i); }, [](const Key& k) { return k.second; });
  }
  if (completed != n) {
    kvpr::set_error("%lld of %lld tasks never became ready", n - completed, n);
    return KVPR_ECYCLE;
  }
  return KVPR_OK;
}

}  // extern "C"
