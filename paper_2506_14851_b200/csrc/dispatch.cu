// K6: dispatch / preemption plan over the task queues of the slot backends
// (SURVEY.md 8(f) row 2): the consumer of the priority keys.
//
// Reference (pdgsim/simcore.py): on every PriorityRefresh (636-644) the
// simulator preempts on every backend (_preempt, 652-687) and then fills free
// slots (_dispatch, 512-516).  Both pick tasks by _task_sort_key (339-344):
// the tuple (priority key, arrival_time, app_instance_id, stage_index,
// request_index), a total order.  _dispatch starts min(queue) while a slot is
// free; _preempt repeatedly compares w = min(queue) with x = max(active) and
// swaps them while x.key > w.key * hysteresis and x.key > w.key.
//
// Device mapping: one stable LSD radix sort of all tasks by (backend, key,
// app arrival rank, stage, request) -- three CUB passes over 64-bit keys --
// gives every backend a segment in tuple order, so "min"/"max" become
// positions.  One CTA per backend then compacts, in order, the segment's
// running tasks (all of them) and its first 2*slots waiting tasks (no plan
// can start more), and one thread replays the reference loops on those short
// lists in shared memory, emitting the events (preempt / start) in the order
// the simulator applies them.
#include <cooperative_groups.h>

#include <algorithm>


#include "common.cuh"

namespace pdg {

constexpr int kPlanThreads = 256;
constexpr int kMaxSlots = 1024;

__device__ __forceinline__ uint64_t orderable_u64(double x) {
  const uint64_t b = uint64_t(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void tie_keys_kernel(const uint32_t* __restrict__ app_rank,
                                const int32_t* __restrict__ stage,
                                const int32_t* __restrict__ request, int64_t n,
                                uint64_t* __restrict__ k, uint32_t* __restrict__ idx) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x) {
    k[t] = (uint64_t(app_rank[t]) << 32) | (uint64_t(uint32_t(stage[t]) & 0xffffu) << 16) |
           (uint64_t(uint32_t(request[t]) & 0xffffu));
    idx[t] = uint32_t(t);
  }
}

__global__ void gather_key_kernel(const double* __restrict__ key,
                                  const uint32_t* __restrict__ idx, int64_t n,
                                  uint64_t* __restrict__ k) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    k[i] = orderable_u64(key[idx[i]]);
}

__global__ void gather_backend_kernel(const int32_t* __restrict__ backend,
                                      const uint32_t* __restrict__ idx, int64_t n,
                                      uint64_t* __restrict__ k, int32_t* __restrict__ count) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t b = backend[idx[i]];
    k[i] = uint64_t(uint32_t(b));
    atomicAdd(count + b, 1);
  }
}

struct PlanArgs {
  const uint32_t* order;       // [n] task ids in (backend, tuple) order
  const int32_t* count;        // [nb] tasks per backend
  const uint8_t* active;       // [n] by task id
  const double* key;           // [n] by task id
  const int32_t* slots;        // [nb]
  int32_t nb;
  double hysteresis;
  int32_t preempt;
  int32_t ev_cap;              // events per backend
  int32_t* ev_task;            // [nb, ev_cap]
  uint8_t* ev_kind;            // [nb, ev_cap]
  int32_t* ev_count;           // [nb]
  int32_t* status;             // [1] 0 ok, 1 more running tasks than slots
};

// ordered compaction of one predicate over a chunk (block-wide)
__device__ __forceinline__ int block_rank(bool p, int& total, int* warp_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(kFull, p);
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  if (lane == 0) warp_tot[wid] = __popc(b);
  __syncthreads();
  int before = 0, tot = 0;
  for (int w = 0; w < kPlanThreads / 32; ++w) {
    before += w < wid ? warp_tot[w] : 0;
    tot += warp_tot[w];
  }
  __syncthreads();
  total = tot;
  return before + __popc(b & lt);
}

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(PlanArgs a) {
  __shared__ int s_act[kMaxSlots + 1];
  __shared__ int s_q[2 * kMaxSlots];
  __shared__ int s_pre[kMaxSlots + 1];
  __shared__ int warp_tot[kPlanThreads / 32];
  __shared__ int s_off;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    int off = 0;
    for (int i = 0; i < b; ++i) off += a.count[i];
    s_off = off;
  }
  __syncthreads();
  const int start = s_off, len = a.count[b];
  const int slots = a.slots[b];
  const int qcap = 2 * slots;
  int na = 0, nq = 0;
  for (int base = 0; base < len; base += kPlanThreads) {
    const int p = base + threadIdx.x;
    const bool in = p < len;
    const uint32_t t = in ? a.order[start + p] : 0u;
    const bool act = in && a.active[t];
    int tot;
    const int ra = block_rank(act, tot, warp_tot);
    if (act && na + ra <= kMaxSlots) s_act[na + ra] = p;
    na += tot;
    const int rq = block_rank(in && !act, tot, warp_tot);
    if (in && !act && nq + rq < qcap) s_q[nq + rq] = p;
    nq = min(nq + tot, qcap);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int* evt = a.ev_task + size_t(b) * a.ev_cap;
  uint8_t* evk = a.ev_kind + size_t(b) * a.ev_cap;
  int ne = 0;
  if (na > slots) {                             // the simulator never lets this happen
    atomicExch(a.status, 1);
    a.ev_count[b] = 0;
    return;
  }
  auto key_at = [&](int p) { return a.key[a.order[start + p]]; };
  auto task_at = [&](int p) { return int32_t(a.order[start + p]); };
  // active: s_act ascending (max = last); waiting: s_q[qi..] merged with the
  // preempted tasks s_pre (ascending)
  int qi = 0, np = 0;
  const bool truncated = len - na > nq;         // waiting tasks beyond the candidates
  auto wait_min = [&](bool take) -> int {
    if (qi == nq && truncated) {                // would need a task past the list
      atomicExch(a.status, 2);
      return -1;
    }
    const bool fromq = qi < nq && (np == 0 || s_q[qi] < s_pre[0]);
    if (!fromq && np == 0) return -1;
    const int p = fromq ? s_q[qi] : s_pre[0];
    if (take) {
      if (fromq) {
        ++qi;
      } else {
        for (int i = 1; i < np; ++i) s_pre[i - 1] = s_pre[i];
        --np;
      }
    }
    return p;
  };
  auto insert_sorted = [&](int* arr, int& n, int p) {
    int i = n++;
    while (i > 0 && arr[i - 1] > p) {
      arr[i] = arr[i - 1];
      --i;
    }
    arr[i] = p;
  };
  if (a.preempt) {                              // _preempt (simcore.py:652-687)
    for (;;) {
      if (na == 0) break;
      const int w = wait_min(false);
      if (w < 0) break;
      const int x = s_act[na - 1];
      const double wk = key_at(w), xk = key_at(x);
      if (!(xk > __dmul_rn(wk, a.hysteresis) && xk > wk)) break;
      wait_min(true);
      --na;                                     // x leaves the slots ...
      insert_sorted(s_pre, np, x);              // ... and waits again
      insert_sorted(s_act, na, w);
      if (ne + 2 <= a.ev_cap) {
        evt[ne] = task_at(x); evk[ne] = 1;      // preempt x
        evt[ne + 1] = task_at(w); evk[ne + 1] = 2;   // start w
      }
      ne += 2;
    }
  }
  a.ev_count[b] = ne;                           // preempt events of this backend
  int nd = 0;                                   // then its dispatch events
  while (na < slots) {                          // _dispatch (simcore.py:512-516)
    const int w = wait_min(true);
    if (w < 0) break;
    ++na;
    if (ne + nd < a.ev_cap) {
      evt[ne + nd] = task_at(w);
      evk[ne + nd] = 2;
    }
    ++nd;
  }
  a.ev_count[a.nb + b] = nd;
}

}  // namespace pdg

using namespace pdg;

extern "C" size_t pdg_dispatch_temp_bytes(int64_t n, int32_t n_backends) {
  const size_t sort_tmp = order_temp_bytes(n > 0 ? n : 1);
  const size_t nn = size_t(n > 0 ? n : 1);
  // keys x2 (u64), idx x2 (u32), counts (nb), status, sort temp
  return 2 * nn * 8 + 2 * nn * 4 + size_t(n_backends) * 4 + 256 + sort_tmp + 1024;
}

extern "C" int pdg_dispatch_plan(const int32_t* backend, const uint8_t* active,
                                 const double* key, const uint32_t* app_rank,
                                 const int32_t* stage, const int32_t* request, int64_t n,
                                 const int32_t* slots, int32_t n_backends, double hysteresis,
                                 int32_t preempt, int32_t ev_cap, int32_t* ev_task,
                                 uint8_t* ev_kind, int32_t* ev_count, void* temp,
                                 size_t temp_bytes, void* stream) {
  if (n < 0 || n > INT32_MAX || n_backends < 1 || n_backends > 65535 || ev_cap < 0 ||
      (n > 0 && (!backend || !active || !key || !app_rank || !stage || !request)) || !slots ||
      !ev_task || !ev_kind || !ev_count || !temp) {
    set_error("pdg_dispatch_plan: invalid arguments");
    return PDG_EINVAL;
  }
  const size_t need = pdg_dispatch_temp_bytes(n, n_backends);
  if (temp_bytes < need) {
    set_error("pdg_dispatch_plan: temp_bytes %zu < %zu", temp_bytes, need);
    return PDG_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nn = size_t(n > 0 ? n : 1);
  char* p = static_cast<char*>(temp);
  uint64_t* k0 = reinterpret_cast<uint64_t*>(p);
  uint64_t* k1 = k0 + nn;
  uint32_t* i0 = reinterpret_cast<uint32_t*>(k1 + nn);
  uint32_t* i1 = i0 + nn;
  int32_t* count = reinterpret_cast<int32_t*>(i1 + nn);
  int32_t* status = count + n_backends;
  char* sort_tmp = reinterpret_cast<char*>(
      (reinterpret_cast<uintptr_t>(status + 64) + 255) & ~uintptr_t(255));
  size_t sort_bytes = temp_bytes - size_t(sort_tmp - p);
  cudaError_t e = cudaMemsetAsync(count, 0, size_t(n_backends) * 4 + 4, st);
  if (e != cudaSuccess) return cuda_status(e, "pdg_dispatch_plan memset");
  e = cudaMemsetAsync(ev_count, 0, size_t(2 * n_backends) * 4, st);
  if (e != cudaSuccess) return cuda_status(e, "pdg_dispatch_plan memset");
  if (n > 0) {
    const int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > int64_t(sm_count()) * 8) blocks = int64_t(sm_count()) * 8;
    tie_keys_kernel<<<unsigned(blocks), threads, 0, st>>>(app_rank, stage, request, n, k0, i0);
    // LSD: tie-break fields, then the priority key, then the backend (stable)
    if (int r = order_sort(k0, k1, i0, i1, n, 0, 64, sort_tmp, sort_bytes, st)) return r;
    gather_key_kernel<<<unsigned(blocks), threads, 0, st>>>(key, i1, n, k0);
    if (int r = order_sort(k0, k1, i1, i0, n, 0, 64, sort_tmp, sort_bytes, st)) return r;
    gather_backend_kernel<<<unsigned(blocks), threads, 0, st>>>(backend, i0, n, k0, count);
    int bits = 1;
    while ((1 << bits) < n_backends) ++bits;
    if (int r = order_sort(k0, k1, i0, i1, n, 0, bits, sort_tmp, sort_bytes, st)) return r;
  }
  PlanArgs a{i1, count, active, key, slots, n_backends, hysteresis, preempt, ev_cap,
             ev_task, ev_kind, ev_count, status};
  plan_kernel<<<unsigned(n_backends), kPlanThreads, 0, st>>>(a);
  return launch_status("plan_kernel");
}

extern "C" int pdg_dispatch_status(const void* temp, int64_t n, int32_t n_backends,
                                   int32_t* status_out, void* stream) {
  if (!temp || !status_out || n_backends < 1) {
    set_error("pdg_dispatch_status: invalid arguments");
    return PDG_EINVAL;
  }
  const size_t nn = size_t(n > 0 ? n : 1);
  const char* p = static_cast<const char*>(temp);
  const int32_t* status = reinterpret_cast<const int32_t*>(p + 2 * nn * 8 + 2 * nn * 4) +
                          n_backends;
  return cuda_status(cudaMemcpyAsync(status_out, status, 4, cudaMemcpyDeviceToHost,
                                     (cudaStream_t)stream),
                     "pdg_dispatch_status");
}

// ---------------------------------------------------------------------------
// a11b: Simulator._update_attained (simcore.py:306-313) for a whole queue.
// age[a] = completed[a] + max(progress[a], max over active started tasks t of
// app a of min(service[t], max(0, now - (start[t] + cold[t])))).  The max is
// taken with 64-bit atomicMax on order-preserving images of the doubles, so
// the result does not depend on task order: bit-identical to the reference
// loop (which returns the first of equal values; only +0/-0 could differ).
// ---------------------------------------------------------------------------
#ifndef PDG_ATTAINED_FUSED
#define PDG_ATTAINED_FUSED 1
#endif
namespace pdg {
constexpr bool kAttainedFused = PDG_ATTAINED_FUSED != 0;
__device__ __forceinline__ double from_orderable_u64(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

__global__ void attained_init_kernel(const double* __restrict__ progress, int64_t n,
                                     uint64_t* __restrict__ best) {
  for (int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; a < n;
       a += int64_t(gridDim.x) * blockDim.x)
    best[a] = orderable_u64(progress[a]);
}

__global__ void attained_tasks_kernel(const int32_t* __restrict__ app,
                                      const uint8_t* __restrict__ active,
                                      const double* __restrict__ start,
                                      const double* __restrict__ cold,
                                      const double* __restrict__ service, int64_t n_tasks,
                                      int64_t n_apps, double now, uint64_t* __restrict__ best) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n_tasks;
       t += int64_t(gridDim.x) * blockDim.x) {
    const double st = start[t];
    const int32_t a = app[t];
    if (!active[t] || st != st || a < 0 || a >= n_apps) continue;  // not running / not started
    const double x = dsub(now, dadd(st, cold[t]));
    const double run = x > 0.0 ? x : 0.0;                         // max(0.0, x)
    const double sv = service[t];
    const double v = run < sv ? run : sv;                         // min(service, run)
    atomicMax(reinterpret_cast<unsigned long long*>(best + a),
              static_cast<unsigned long long>(orderable_u64(v)));
  }
}

__global__ void attained_final_kernel(const double* __restrict__ completed,
                                      const uint64_t* __restrict__ best, int64_t n,
                                      double* __restrict__ age) {
  for (int64_t a = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; a < n;
       a += int64_t(gridDim.x) * blockDim.x)
    age[a] = dadd(completed[a], from_orderable_u64(best[a]));
}
// the three phases in ONE cooperative kernel (grid barriers instead of two
// kernel boundaries): init -> task maxima -> final sum
__global__ void __launch_bounds__(256) attained_fused_kernel(
    const double* __restrict__ completed, const double* __restrict__ progress, int64_t n,
    const int32_t* __restrict__ app, const uint8_t* __restrict__ active,
    const double* __restrict__ start, const double* __restrict__ cold,
    const double* __restrict__ service, int64_t n_tasks, double now, uint64_t* best,
    double* __restrict__ age) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t a = i0; a < n; a += stride) best[a] = orderable_u64(progress[a]);
  if (n_tasks > 0) {
    grid.sync();
    for (int64_t t = i0; t < n_tasks; t += stride) {
      const double st = start[t];
      const int32_t a = app[t];
      if (!active[t] || st != st || a < 0 || a >= n) continue;
      const double x = dsub(now, dadd(st, cold[t]));
      const double run = x > 0.0 ? x : 0.0;
      const double sv = service[t];
      const double v = run < sv ? run : sv;
      atomicMax(reinterpret_cast<unsigned long long*>(best + a),
                static_cast<unsigned long long>(orderable_u64(v)));
    }
  }
  grid.sync();
  for (int64_t a = i0; a < n; a += stride)
    age[a] = dadd(completed[a], from_orderable_u64(__ldcg(best + a)));
}
}  // namespace pdg

extern "C" int pdg_attained_service(const double* completed, const double* progress,
                                    int64_t n_apps, const int32_t* task_app,
                                    const uint8_t* task_active, const double* task_start,
                                    const double* task_cold, const double* task_service,
                                    int64_t n_tasks, double now, double* age_out, void* temp,
                                    size_t temp_bytes, void* stream) {
  if (n_apps < 0 || n_tasks < 0 ||
      (n_apps > 0 && (!completed || !progress || !age_out || !temp)) ||
      (n_tasks > 0 && (!task_app || !task_active || !task_start || !task_cold ||
                       !task_service))) {
    set_error("pdg_attained_service: invalid arguments");
    return PDG_EINVAL;
  }
  if (n_apps == 0) return PDG_OK;
  if (temp_bytes < size_t(n_apps) * 8) {
    set_error("pdg_attained_service: temp_bytes %zu < %lld", temp_bytes,
              (long long)(n_apps * 8));
    return PDG_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t* best = static_cast<uint64_t*>(temp);
  if (kAttainedFused) {
    int per_sm = 0;
    if (int r = launch_setup(reinterpret_cast<const void*>(attained_fused_kernel), 256, 0,
                             &per_sm))
      return r;
    const int64_t m = std::max(n_apps, n_tasks);
    const int64_t g = std::min<int64_t>((m + 255) / 256, int64_t(per_sm) * sm_count());
    void* args[] = {&completed, &progress, &n_apps, &task_app, &task_active, &task_start,
                    &task_cold, &task_service, &n_tasks, &now, &best, &age_out};
    return cuda_status(cudaLaunchCooperativeKernel(
                           reinterpret_cast<const void*>(attained_fused_kernel),
                           dim3(unsigned(g)), dim3(256), args, 0, st),
                       "attained_fused_kernel");
  }
  const int64_t cap = int64_t(sm_count()) * 8;
  auto grid = [&](int64_t m) { return unsigned(std::min<int64_t>((m + 255) / 256, cap)); };
  attained_init_kernel<<<grid(n_apps), 256, 0, st>>>(progress, n_apps, best);
  int rc = launch_status("attained_init_kernel");
  if (rc != PDG_OK) return rc;
  if (n_tasks > 0) {
    attained_tasks_kernel<<<grid(n_tasks), 256, 0, st>>>(task_app, task_active, task_start,
                                                         task_cold, task_service, n_tasks,
                                                         n_apps, now, best);
    rc = launch_status("attained_tasks_kernel");
    if (rc != PDG_OK) return rc;
  }
  attained_final_kernel<<<grid(n_apps), 256, 0, st>>>(completed, best, n_apps, age_out);
  return launch_status("attained_final_kernel");
}
