// abi.cpp — the C ABI of libleyenda.so (include/leyenda.h): validation, pointer classification,
// path dispatch ("adaptive ... internal or external sort"),
// per-device serialisation and error reporting.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "config.h"
#include "leyenda.h"
#include "runtime.h"

namespace ley {
ley_status sort_external_host(DeviceContext& ctx, const uint8_t* in, uint8_t* out, uint32_t* perm_out, uint64_t n,
                              uint64_t budget, uint32_t key_bytes, cudaStream_t s, Profiler& prof);
ley_status dist_sort(ley_comm* comm, const void* in_local, uint64_t n_local, void* out_local, uint64_t out_capacity,
                     uint64_t* n_out_local, uint64_t* out_global_offset, uint64_t budget, uint32_t key_bytes,
                     cudaStream_t s);
ley_status comm_get_unique_id(uint8_t id_out[128]);
ley_status comm_init(ley_comm** comm, int nranks, int rank, const uint8_t id[128], int device);
ley_status comm_destroy(ley_comm* comm);
ley_status dist_sort_loopback(int G, const void* const* in, const uint64_t* n_local, void* const* out,
                              const uint64_t* caps, uint64_t* n_out, uint64_t* out_off, uint64_t budget,
                              uint32_t key_bytes, cudaStream_t s);
int dist_plan_splitters(const uint64_t* hist, uint64_t N, int G, uint32_t* bins, uint64_t* rho, uint64_t* first);
ley_status test_shared_scratch(const char* name, uint64_t bytes, int create, void** ptr);
void test_shared_scratch_close(void* p, uint64_t bytes, const char* unlink_name);
void dist_bin_dest_counts(const uint64_t* local_hist, const uint32_t* bins, int nspl, uint64_t* counts);
void dist_plan_exchange(const uint64_t* send_counts, int G, int rank, uint64_t* recv_counts, uint64_t* recv_off,
                        uint64_t* send_off, uint64_t* n_out, uint64_t* out_off);
void dist_dest_offsets(const uint64_t* send_counts, int G, int rank, uint64_t* dst_off);
}  // namespace ley

using namespace ley;

namespace {

enum class Kind { kDevice, kPinnedHost, kOther };

ley_status classify_ptr(const void* p, int cur_dev, Kind* kind, const char* what) {
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("validate: cudaPointerGetAttributes(") + what + ") failed: " + cudaGetErrorString(e));
    return LEY_ERR_CUDA;
  }
  switch (a.type) {
    case cudaMemoryTypeDevice:
      if (a.device != cur_dev) {
        set_error(std::string("validate: ") + what + " lives on device " + std::to_string(a.device) +
                  " but the current device is " + std::to_string(cur_dev));
        return LEY_ERR_INVALID_ARGUMENT;
      }
      *kind = Kind::kDevice;
      return LEY_OK;
    case cudaMemoryTypeHost:
      *kind = Kind::kPinnedHost;
      return LEY_OK;
    default:
      *kind = Kind::kOther;
      set_error(std::string("validate: ") + what +
                " is pageable or managed memory; pass device memory or pinned host memory");
      return LEY_ERR_UNSUPPORTED;
  }
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
  return x < y + nb && y < x + na;
}

// Records are 100 bytes. Keys: record bytes [0, key_bytes), 1 <= key_bytes <= 100 — the paper's
// 10 and its "flexible key sizes".
ley_status check_record_key(uint32_t rb, uint32_t kb, uint32_t max_kb) {
  if (rb != kRecordBytes || kb < 1 || kb > max_kb) {
    set_error("validate: record_bytes must be 100 and key_bytes 1.." + std::to_string(max_kb) + " on this path (P:126, P:164)");
    return LEY_ERR_UNSUPPORTED;
  }
  return LEY_OK;
}

ley_status check_common(const void* in, const void* out, const void* perm, uint64_t n, uint32_t rb, uint32_t kb) {
  if (ley_status st = check_record_key(rb, kb, kRecordBytes)) return st;
  if (n == 0) return LEY_OK;
  if (n > LEY_MAX_RECORDS) {
    set_error("validate: n_records > 2^32-2 (u32 ordinals)");
    return LEY_ERR_TOO_LARGE;
  }
  if (!in || !out) {
    set_error("validate: NULL in/out with n_records > 0");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  if (((uintptr_t)in & 15) || ((uintptr_t)out & 15) || ((uintptr_t)perm & 3)) {
    set_error("validate: in/out must be 16-byte aligned (perm 4-byte aligned)");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  const size_t bytes = (size_t)n * kRecordBytes;
  if (overlaps(in, bytes, out, bytes) || (perm && (overlaps(perm, 4 * n, out, bytes) || overlaps(perm, 4 * n, in, bytes)))) {
    set_error("validate: in, out and perm must not overlap (out-of-place sort)");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  return LEY_OK;
}

}  // namespace

extern "C" {

const char* ley_last_error(void) { return last_error(); }

uint32_t ley_version(void) { return (1u << 16) | 1u; }  // 1.1: key_bytes 1..100, host path 2

ley_status ley_set_option(const char* name, int64_t value) {
  clear_error();
  return option_set(name, value);
}

ley_status ley_get_option(const char* name, int64_t* value) {
  clear_error();
  return option_get(name, value);
}

ley_status ley_plan_query(uint64_t n_records, uint64_t device_budget_bytes, ley_plan_info* info) {
  clear_error();
  return plan_query(n_records, device_budget_bytes, info);
}

int ley_stage_times(const char** names, float* ms, int max, int* launches) {
  return stage_times(names, ms, max, launches);
}

ley_status ley_device_bytes(uint64_t* current_bytes, uint64_t* peak_bytes, int reset_peak) {
  clear_error();
  device_bytes(current_bytes, peak_bytes, reset_peak != 0);
  return LEY_OK;
}

ley_status ley_release_cache(int device) {
  clear_error();
  release_device(device);
  return LEY_OK;
}

ley_status ley_sort_perm(const void* in, void* out, uint32_t* perm, uint64_t n_records, uint32_t record_bytes,
                         uint32_t key_bytes, uint64_t device_budget_bytes, void* stream) {
  clear_error();
  record_launches(0);
  ley_status st = check_common(in, out, perm, n_records, record_bytes, key_bytes);
  if (st || n_records == 0) return st;
  int dev = 0;
  {
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error(std::string("validate: no CUDA device (") + cudaGetErrorString(e) + ")");
      return LEY_ERR_CUDA;
    }
  }
  Kind kin, kout, kperm = Kind::kDevice;
  if ((st = classify_ptr(in, dev, &kin, "in"))) return st;
  if ((st = classify_ptr(out, dev, &kout, "out"))) return st;
  if (perm && (st = classify_ptr(perm, dev, &kperm, "perm"))) return st;
  if (kin != kout || (perm && kperm != kout)) {
    set_error("validate: in, out (and perm) must be the same memory kind (all device or all pinned host)");
    return LEY_ERR_UNSUPPORTED;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceContext& ctx = device_context(dev);
  std::lock_guard<std::mutex> guard(ctx.mu);
  if (ctx.device != dev || ctx.sms <= 0) ctx.device = dev;
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms > 0) ctx.sms = sms;
  }
  const Options opts = options_snapshot();
  if ((st = async_join(ctx, s))) return st;  // (a previous stream-ordered sort may still use the buffers)
  if (opts.l2_fetch_bytes) LEY_CUDA("setup", cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)opts.l2_fetch_bytes));
  Profiler prof;
  prof.on = opts.profile != 0;
  prof.stream = s;
  prof.ctx = &ctx;
  const uint8_t* in8 = static_cast<const uint8_t*>(in);
  uint8_t* out8 = static_cast<uint8_t*>(out);

  if (kin == Kind::kDevice) {
    InternalLayout L = plan_internal(n_records);
    const uint64_t need = L.bytes + internal_aux_bytes(n_records) + keypass_bytes(n_records, key_bytes, perm != nullptr);
    if (device_budget_bytes && need > device_budget_bytes) {
      set_error("plan: internal path needs " + std::to_string(need) + " bytes of device scratch, budget is " +
                std::to_string(device_budget_bytes));
      return LEY_ERR_BUDGET;
    }
    st = sort_internal_device(ctx, in8, out8, perm, n_records, s, prof, nullptr, 0, key_bytes, opts.async != 0);
  } else {
    ley_plan_info info;
    plan_query(n_records, device_budget_bytes, &info);
    if (key_bytes > kKeyBytes) {  // multi-pass keys: the staged path only (it needs a device output)
      const uint64_t need = info.staged_bytes + keypass_bytes(n_records, key_bytes, perm != nullptr);
      if (device_budget_bytes && need > device_budget_bytes) {
        set_error("plan: keys longer than 10 bytes on host pointers take the staged path, which needs " +
                  std::to_string(need) + " device bytes; budget is " + std::to_string(device_budget_bytes));
        return LEY_ERR_UNSUPPORTED;
      }
      info.host_path = 0;
    }
    if (info.host_path == 0) {
      // staged internal: H2D, internal sort, D2H
      const size_t bytes = (size_t)n_records * kRecordBytes;
      const size_t a = (bytes + 255) & ~size_t(255);
      if ((st = ensure_buffer(ctx.stage, 2 * a, "staging", s))) return st;
      uint8_t* din = static_cast<uint8_t*>(ctx.stage.ptr);
      uint8_t* dout = din + a;
      if ((st = prof.begin("H2D"))) return st;
      LEY_CUDA("H2D", cudaMemcpyAsync(din, in8, bytes, cudaMemcpyHostToDevice, s));
      if ((st = prof.end())) return st;
      st = sort_internal_device(ctx, din, dout, perm, n_records, s, prof, nullptr, 0, key_bytes);
      if (st) return st;
      if ((st = prof.begin("D2H"))) return st;
      if ((st = copy_split(ctx, out8, dout, bytes, cudaMemcpyDeviceToHost, s, DeviceContext::kSplitParts))) return st;
      if ((st = prof.end())) return st;
    } else if (info.host_path == 2) {
      st = sort_resident_host(ctx, in8, out8, perm, n_records, key_bytes, s, prof);
    } else {
      st = sort_external_host(ctx, in8, out8, perm, n_records, device_budget_bytes, key_bytes, s, prof);
    }
  }
  if (st) return st;
  if (ctx.async_pending) {  // stream-ordered: out is complete when the stream gets there
    record_launches(prof.launches);
    return LEY_OK;
  }
  LEY_CUDA("complete", cudaStreamSynchronize(s));
  LEY_CUDA("complete", cudaGetLastError());
  prof.finish();
  return LEY_OK;
}

ley_status ley_sort(const void* in, void* out, uint64_t n_records, uint32_t record_bytes, uint32_t key_bytes,
                    uint64_t device_budget_bytes, void* stream) {
  return ley_sort_perm(in, out, nullptr, n_records, record_bytes, key_bytes, device_budget_bytes, stream);
}

ley_status ley_sort_submit(const void* in, void* out, uint64_t n_records, uint32_t record_bytes, uint32_t key_bytes,
                           uint64_t device_budget_bytes, void* stream) {
  clear_error();
  record_launches(0);
  ley_status st = check_common(in, out, nullptr, n_records, record_bytes, key_bytes);
  if (st || n_records == 0) return st;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    set_error("validate: no CUDA device");
    return LEY_ERR_CUDA;
  }
  Kind kin, kout;
  if ((st = classify_ptr(in, dev, &kin, "in"))) return st;
  if ((st = classify_ptr(out, dev, &kout, "out"))) return st;
  if (kin != Kind::kPinnedHost || kout != Kind::kPinnedHost) {
    set_error("validate: ley_sort_submit takes pinned host in/out (device buffers: call ley_sort)");
    return LEY_ERR_UNSUPPORTED;
  }
  const size_t a = ((size_t)n_records * kRecordBytes + 255) & ~size_t(255);
  const uint64_t need = 4 * (uint64_t)a + plan_internal(n_records).bytes +  // two slots (in | out) + scratch
                        keypass_bytes(n_records, key_bytes, false);
  if (device_budget_bytes && need > device_budget_bytes)  // does not fit twice: the blocking path decides
    return ley_sort(in, out, n_records, record_bytes, key_bytes, device_budget_bytes, stream);
  DeviceContext& ctx = device_context(dev);  // (device index and SM count are set on creation)
  // the pipeline has its own lock; its worker takes ctx.mu for each sort. Not taking ctx.mu here keeps a
  // submit from waiting for the previous call's sort to finish.
  return sort_submit(ctx, static_cast<const uint8_t*>(in), static_cast<uint8_t*>(out), n_records, key_bytes,
                     static_cast<cudaStream_t>(stream));
}

ley_status ley_sort_drain(void) {
  clear_error();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    set_error("validate: no CUDA device");
    return LEY_ERR_CUDA;
  }
  DeviceContext& ctx = device_context(dev);
  return sort_drain(ctx);
}

ley_status ley_comm_get_unique_id(uint8_t id_out[128]) {
  clear_error();
  return comm_get_unique_id(id_out);
}

ley_status ley_comm_init(ley_comm** comm, int nranks, int rank, const uint8_t id[128], int device) {
  clear_error();
  return comm_init(comm, nranks, rank, id, device);
}

ley_status ley_sort_dist(ley_comm* comm, const void* in_local, uint64_t n_local, void* out_local,
                         uint64_t out_capacity_records, uint64_t* n_out_local, uint64_t* out_global_offset,
                         uint32_t record_bytes, uint32_t key_bytes, uint64_t device_budget_bytes, void* stream) {
  clear_error();
  if (ley_status st = check_record_key(record_bytes, key_bytes, kKeyBytes)) return st;
  if (!comm || !n_out_local || !out_global_offset) {
    set_error("validate: NULL comm / n_out_local / out_global_offset");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  return dist_sort(comm, in_local, n_local, out_local, out_capacity_records, n_out_local, out_global_offset,
                   device_budget_bytes, key_bytes, static_cast<cudaStream_t>(stream));
}

ley_status ley_comm_destroy(ley_comm* comm) {
  clear_error();
  return comm_destroy(comm);
}

ley_status ley_sort_dist_loopback(int nranks, const void* const* in_local, const uint64_t* n_local,
                                  void* const* out_local, const uint64_t* out_capacity_records, uint64_t* n_out_local,
                                  uint64_t* out_global_offset, uint32_t record_bytes, uint32_t key_bytes,
                                  uint64_t device_budget_bytes, void* stream) {
  clear_error();
  if (ley_status st = check_record_key(record_bytes, key_bytes, kKeyBytes)) return st;
  if (!in_local || !n_local || !out_local || !out_capacity_records || !n_out_local || !out_global_offset) {
    set_error("validate: NULL argument array");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  return dist_sort_loopback(nranks, in_local, n_local, out_local, out_capacity_records, n_out_local,
                            out_global_offset, device_budget_bytes, key_bytes, static_cast<cudaStream_t>(stream));
}

int ley_dist_plan_splitters(const uint64_t* global_hist16, uint64_t n_total, int nranks, uint32_t* bins,
                            uint64_t* rank_in_bin, uint64_t* bin_first) {
  if (!global_hist16 || !bins || !rank_in_bin || !bin_first) return 1;
  return dist_plan_splitters(global_hist16, n_total, nranks, bins, rank_in_bin, bin_first);
}

void ley_dist_bin_dest_counts(const uint64_t* local_hist16, const uint32_t* bins, int nranks, uint64_t* counts) {
  dist_bin_dest_counts(local_hist16, bins, nranks - 1, counts);
}

void ley_dist_plan_exchange(const uint64_t* send_counts, int nranks, int rank, uint64_t* recv_counts,
                            uint64_t* recv_offsets, uint64_t* send_offsets, uint64_t* n_out, uint64_t* out_offset) {
  dist_plan_exchange(send_counts, nranks, rank, recv_counts, recv_offsets, send_offsets, n_out, out_offset);
}

ley_status ley_test_shared_scratch(const char* name, uint64_t bytes, int create, void** ptr) {
  clear_error();
  if (!name || !ptr) {
    set_error("ley_test_shared_scratch: NULL");
    return LEY_ERR_INVALID_ARGUMENT;
  }
  return test_shared_scratch(name, bytes, create, ptr);
}

void ley_test_shared_scratch_close(void* ptr, uint64_t bytes, const char* unlink_name) {
  test_shared_scratch_close(ptr, bytes, unlink_name);
}

void ley_dist_dest_offsets(const uint64_t* send_counts, int nranks, int rank, uint64_t* dst_offsets) {
  dist_dest_offsets(send_counts, nranks, rank, dst_offsets);
}

}  // extern "C"
