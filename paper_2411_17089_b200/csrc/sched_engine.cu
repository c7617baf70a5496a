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
  std::vector<long long> indeg(n);
  std::vector<std::vector<long long>> children(n);
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
      children[d].push_back(i);
    }
  }
  using Key = std::pair<long long, long long>;  // (priority, id): Python's heapq order on tuples
  std::vector<std::priority_queue<Key, std::vector<Key>, std::greater<Key>>> ready(n_resources);
  for (long long i = 0; i < n; ++i)
    if (indeg[i] == 0) ready[resource[i]].push({priority[i], i});
  std::vector<long long> running_id(n_resources, -1);
  std::vector<double> running_end(n_resources, 0.0);
  long long completed = 0;
  auto dispatch = [&](double now) {
    for (int r = 0; r < n_resources; ++r) {
      if (running_id[r] < 0 && !ready[r].empty()) {
        const long long i = ready[r].top().second;
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
        for (long long c : children[i])
          if (--indeg[c] == 0) ready[resource[c]].push({priority[c], c});
      }
    }
    dispatch(t);
  }
  if (completed != n) {
    kvpr::set_error("%lld of %lld tasks never became ready", n - completed, n);
    return KVPR_ECYCLE;
  }
  return KVPR_OK;
}

}  // extern "C"
