// abi.cu -- C-ABI plumbing (errors, stats, device info) and the host-buffer
// entry point mckg_detect_shared_host, which streams a host-resident trace to
// the device in chunks on two CUDA streams so that the PCIe copies of chunk
// c+1 overlap the detection of chunk c.
#include <array>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace mckg {

namespace {
thread_local std::string g_err;
thread_local mckg_launch_stats g_stats{};
}  // namespace

void set_error(const char* what, cudaError_t e) {
  g_err = what;
  if (e != cudaSuccess) {
    g_err += ": ";
    g_err += cudaGetErrorString(e);
  }
}

void note_launch(uint32_t kernels, uint32_t grid, uint32_t block, uint32_t smem) {
  g_stats.kernels = kernels;
  g_stats.grid = grid;
  g_stats.block = block;
  g_stats.smem_bytes = smem;
}

void add_launches(uint32_t kernels) { g_stats.kernels = kernels; }

// Experiment / test switches (MCKG_DEBUG at load time, mckg_set_debug later).
static std::atomic<uint32_t>& debug_word() {
  static std::atomic<uint32_t> w{[] {
    const char* e = getenv("MCKG_DEBUG");
    return e ? (uint32_t)atoi(e) : 0u;
  }()};
  return w;
}
uint32_t debug_flags() { return debug_word().load(std::memory_order_relaxed); }

int sm_count() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    if (sms <= 0) sms = 148;
    dev = d;
  }
  return sms;
}

void keep_pool_memory() {
  static thread_local int done_dev = -1;
  int d = 0;
  cudaGetDevice(&d);
  if (d == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done_dev = d;
}

}  // namespace mckg

extern "C" void mckg_set_debug(uint32_t flags) { mckg::debug_word().store(flags); }

using namespace mckg;

extern "C" int mckg_abi_version(void) { return MCKG_ABI_VERSION; }

extern "C" const char* mckg_last_error(void) { return g_err.c_str(); }

extern "C" int mckg_device_count(int* n) {
  if (!n) return MCKG_E_ARG;
  MCKG_CUDA_TRY(cudaGetDeviceCount(n));
  return MCKG_OK;
}

extern "C" int mckg_get_launch_stats(mckg_launch_stats* out) {
  if (!out) return MCKG_E_ARG;
  *out = g_stats;
  return MCKG_OK;
}

extern "C" int mckg_detect_shared_host(const mckg_trace* tr, mckg_race_triple* triples_host,
                                       uint64_t capacity, uint64_t* n_triples_host,
                                       uint64_t* line_first_host, uint32_t* status_host) {
  if (!tr || !n_triples_host || !line_first_host || !status_host ||
      (!triples_host && capacity)) {
    set_error("mckg_detect_shared_host: null argument");
    return MCKG_E_ARG;
  }
  if (tr->n_blocks && (!tr->events || !tr->block_start)) {
    set_error("mckg_detect_shared_host: null trace");
    return MCKG_E_ARG;
  }
  const uint64_t* hbs = tr->block_start;
  // chunk the blocks so each chunk holds <= kChunkEvents records (>= 1 block)
  const uint64_t kChunkEvents = 1ull << 25;  // 512 MiB of records per chunk
  std::vector<uint32_t> cuts{0};
  for (uint32_t b = 0; b < tr->n_blocks;) {
    uint32_t e = b + 1;
    while (e < tr->n_blocks && hbs[e + 1] - hbs[b] <= kChunkEvents) ++e;
    cuts.push_back(e);
    b = e;
  }
  const size_t n_chunks = cuts.size() - 1;
  uint64_t max_ev = 0;
  uint32_t max_nb = 0;
  for (size_t c = 0; c < n_chunks; ++c) {
    max_ev = std::max<uint64_t>(max_ev, hbs[cuts[c + 1]] - hbs[cuts[c]]);
    max_nb = std::max<uint32_t>(max_nb, cuts[c + 1] - cuts[c]);
  }
  // two pipeline streams per device, created once (the detector keeps
  // per-stream scratch, so stable stream handles keep that scratch bounded)
  static std::mutex smu;
  static std::map<int, std::array<cudaStream_t, 2>> sstreams;
  cudaStream_t st[2];
  {
    int dev = 0;
    MCKG_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(smu);
    auto it = sstreams.find(dev);
    if (it == sstreams.end()) {
      std::array<cudaStream_t, 2> a{};
      MCKG_CUDA_TRY(cudaStreamCreateWithFlags(&a[0], cudaStreamNonBlocking));
      MCKG_CUDA_TRY(cudaStreamCreateWithFlags(&a[1], cudaStreamNonBlocking));
      it = sstreams.emplace(dev, a).first;
    }
    st[0] = it->second[0];
    st[1] = it->second[1];
  }
  // device staging, pinned block starts and the outputs are kept per device
  // and grown on demand (large cudaMalloc / cudaMallocHost calls cost
  // milliseconds); one call at a time per device
  struct HostPathScratch {
    std::mutex mu;
    mckg_access* ev[2] = {nullptr, nullptr};
    uint64_t ev_cap = 0;
    uint64_t* bs[2] = {nullptr, nullptr};
    uint64_t bs_cap = 0;
    uint64_t* pin_bs = nullptr;
    uint64_t pin_cap = 0;
    mckg_race_triple* tri = nullptr;
    uint64_t tri_cap = 0;
    unsigned long long* n_tri = nullptr;
    unsigned long long* line_first = nullptr;
    uint32_t* status = nullptr;
  };
  static std::mutex scr_mu;
  static std::map<int, HostPathScratch*> scratch;
  HostPathScratch* S = nullptr;
  {
    int dev = 0;
    MCKG_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(scr_mu);
    HostPathScratch*& e = scratch[dev];
    if (!e) e = new HostPathScratch();
    S = e;
  }
  std::lock_guard<std::mutex> call_lock(S->mu);
  mckg_access* dev_ev[2] = {nullptr, nullptr};
  uint64_t* dev_bs[2] = {nullptr, nullptr};
  uint64_t* pin_bs = nullptr;
  mckg_race_out out{};
  int rc = MCKG_OK;
  uint32_t launches = 0;
  auto fail = [&](const char* what, cudaError_t e) {
    set_error(what, e);
    rc = MCKG_E_CUDA;
  };
  do {
    cudaError_t e;
    const uint64_t need_ev = std::max<uint64_t>(1, max_ev), need_bs = max_nb + 1ull;
    if (S->ev_cap < need_ev) {
      for (int k = 0; k < 2; ++k) {
        cudaFree(S->ev[k]);
        S->ev[k] = nullptr;
      }
      S->ev_cap = 0;
      for (int k = 0; k < 2; ++k)
        if ((e = cudaMalloc(&S->ev[k], need_ev * sizeof(mckg_access)))) break;
      if (e) {
        fail("cudaMalloc(events)", e);
        break;
      }
      S->ev_cap = need_ev;
    }
    if (S->bs_cap < need_bs) {
      for (int k = 0; k < 2; ++k) {
        cudaFree(S->bs[k]);
        S->bs[k] = nullptr;
      }
      S->bs_cap = 0;
      for (int k = 0; k < 2; ++k)
        if ((e = cudaMalloc(&S->bs[k], need_bs * sizeof(uint64_t)))) break;
      if (e) {
        fail("cudaMalloc(block_start)", e);
        break;
      }
      S->bs_cap = need_bs;
    }
    const uint64_t need_pin = tr->n_blocks + n_chunks + 1ull;
    if (S->pin_cap < need_pin) {
      cudaFreeHost(S->pin_bs);
      S->pin_bs = nullptr;
      S->pin_cap = 0;
      if ((e = cudaMallocHost(&S->pin_bs, need_pin * sizeof(uint64_t)))) {
        fail("cudaMallocHost", e);
        break;
      }
      S->pin_cap = need_pin;
    }
    const uint64_t need_tri = std::max<uint64_t>(1, capacity);
    if (S->tri_cap < need_tri) {
      cudaFree(S->tri);
      S->tri = nullptr;
      S->tri_cap = 0;
      if ((e = cudaMalloc(&S->tri, need_tri * sizeof(mckg_race_triple)))) {
        fail("cudaMalloc(triples)", e);
        break;
      }
      S->tri_cap = need_tri;
    }
    if (!S->n_tri) {
      if ((e = cudaMalloc(&S->n_tri, sizeof(unsigned long long))) ||
          (e = cudaMalloc(&S->line_first, MCKG_MAX_LINES * sizeof(unsigned long long))) ||
          (e = cudaMalloc(&S->status, sizeof(uint32_t)))) {
        fail("cudaMalloc(outputs)", e);
        break;
      }
    }
    for (int k = 0; k < 2; ++k) {
      dev_ev[k] = S->ev[k];
      dev_bs[k] = S->bs[k];
    }
    pin_bs = S->pin_bs;
    out.triples = S->tri;
    out.capacity = capacity;
    out.n_triples = S->n_tri;
    out.line_first = S->line_first;
    out.status = S->status;
    if ((rc = mckg_race_out_reset(&out, st[0]))) break;
    ++launches;
    if ((e = cudaStreamSynchronize(st[0]))) {
      fail("reset", e);
      break;
    }
    size_t pos = 0;
    for (size_t c = 0; c < n_chunks && !rc; ++c) {
      const int k = (int)(c & 1);
      const uint32_t b0 = cuts[c], b1 = cuts[c + 1];
      uint64_t* rb = pin_bs + pos;
      for (uint32_t b = b0; b <= b1; ++b) rb[b - b0] = hbs[b] - hbs[b0];
      pos += (b1 - b0) + 1;
      const uint64_t nev = hbs[b1] - hbs[b0];
      if ((e = cudaMemcpyAsync(dev_ev[k], tr->events + hbs[b0], nev * sizeof(mckg_access),
                               cudaMemcpyHostToDevice, st[k]))) {
        fail("cudaMemcpyAsync(events)", e);
        break;
      }
      if ((e = cudaMemcpyAsync(dev_bs[k], rb, (b1 - b0 + 1ull) * sizeof(uint64_t),
                               cudaMemcpyHostToDevice, st[k]))) {
        fail("cudaMemcpyAsync(block_start)", e);
        break;
      }
      mckg_trace sub = *tr;
      sub.events = dev_ev[k];
      sub.block_start = dev_bs[k];
      sub.n_events = nev;
      sub.n_blocks = b1 - b0;
      sub.obj_base = tr->obj_base + b0;
      sub.bid_base = tr->bid_base + b0;
      rc = mckg_detect_shared(&sub, &out, st[k]);
      ++launches;
    }
    if (rc) break;
    if ((e = cudaStreamSynchronize(st[0])) || (e = cudaStreamSynchronize(st[1]))) {
      fail("detect", e);
      break;
    }
    unsigned long long n = 0;
    if ((e = cudaMemcpy(&n, out.n_triples, sizeof n, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(line_first_host, out.line_first, MCKG_MAX_LINES * sizeof(uint64_t),
                        cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(status_host, out.status, sizeof(uint32_t), cudaMemcpyDeviceToHost))) {
      fail("cudaMemcpy(results)", e);
      break;
    }
    if ((*status_host & MCKG_ST_DUP) && n > 0 && n <= capacity) {
      // the per-block dedup set overflowed: restore the exact set on device.
      // (Past capacity the prefix's unique count would understate the total,
      // so the overflow count and the DUP flag are returned as they are.)
      if ((rc = mckg_sort_triples(out.triples, n, tr->obj_base,
                                  out.n_triples, st[0])))
        break;
      launches += 4;
      if ((e = cudaMemcpyAsync(&n, out.n_triples, sizeof n, cudaMemcpyDeviceToHost, st[0])) ||
          (e = cudaStreamSynchronize(st[0]))) {
        fail("dedup", e);
        break;
      }
      *status_host &= ~MCKG_ST_DUP;
    }
    *n_triples_host = n;
    uint64_t nc = std::min<uint64_t>(n, capacity);
    if (nc && (e = cudaMemcpy(triples_host, out.triples, nc * sizeof(mckg_race_triple),
                              cudaMemcpyDeviceToHost))) {
      fail("cudaMemcpy(triples)", e);
      break;
    }
    if (n > capacity) rc = MCKG_E_OVERFLOW;
  } while (0);
  add_launches(launches);
  return rc;
}
