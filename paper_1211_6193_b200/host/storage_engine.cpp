// storage_engine.cpp -- device-memory storage without a GPU.  Used only when
// no CUDA device is present (e.g. the CPU-only test container): cudaMalloc /
// cudaMemcpy / cudaMemset keep working for host-side API checks, and any
// kernel launch fails loudly -- the checker has no CPU execution path for
// device code.
#include <cstring>

#include "engine.hpp"

namespace mckb {
namespace {

class StorageOnlyEngine final : public DeviceEngine {
 public:
  explicit StorageOnlyEngine(std::string why) : why_(std::move(why)) {}
  bool hasDevice() const override { return false; }
  uint64_t alloc(int64_t size) override {
    uint64_t b = bytes_.size();
    bytes_.resize(b + static_cast<size_t>(size), 0);
    meta_.resize(b + static_cast<size_t>(size), 0);
    return b;
  }
  void write(uint64_t base, const uint8_t* b, const uint8_t* m, int64_t n) override {
    std::memcpy(bytes_.data() + base, b, static_cast<size_t>(n));
    std::memcpy(meta_.data() + base, m, static_cast<size_t>(n));
  }
  void read(uint64_t base, uint8_t* b, uint8_t* m, int64_t n) override {
    std::memcpy(b, bytes_.data() + base, static_cast<size_t>(n));
    std::memcpy(m, meta_.data() + base, static_cast<size_t>(n));
  }
  void copy(uint64_t dst, uint64_t src, int64_t n) override {
    std::memmove(bytes_.data() + dst, bytes_.data() + src, static_cast<size_t>(n));
    std::memmove(meta_.data() + dst, meta_.data() + src, static_cast<size_t>(n));
  }
  void fill(uint64_t base, uint8_t v, uint8_t m, int64_t n) override {
    std::memset(bytes_.data() + base, v, static_cast<size_t>(n));
    std::memset(meta_.data() + base, m, static_cast<size_t>(n));
  }
  bool runGrid(const GridSpec&, GridResult& out) override {
    out.error = "no CUDA device (" + why_ + "): device grids run only on the B200 engine";
    return false;
  }

 private:
  std::string why_;
  std::vector<uint8_t> bytes_, meta_;
};

}  // namespace

std::unique_ptr<DeviceEngine> makeStorageOnlyEngine(const std::string& why) {
  return std::unique_ptr<DeviceEngine>(new StorageOnlyEngine(why));
}

}  // namespace mckb
