// dataset.cu -- ATKV dataset container I/O, host and device sides.
//
// Restates the reference's container (dataset.hpp:18-28, dataset.cpp:45-124):
//   bytes 0..3 "ATKV", byte 4 version 1, bytes 5..12 rows u64 LE,
//   bytes 13..20 dims u64 LE, then rows*dims fp32 LE.
// Same checks, same order, same messages (DatasetFormatError -> ATKG_EFORMAT).
//
// B200 side: the device variants stream the payload through two pinned
// staging chunks, so file reads overlap the H2D (or D2H) copies, and the NaN
// rejection runs as an HBM-bound scan kernel on the resident payload instead
// of a host pass.  The payload is raw little-endian fp32, which is the host and
// device byte order, so no per-element swizzle is needed.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "internal.hpp"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "ATKV payloads are little-endian fp32");

namespace atkg {
namespace {

struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };

constexpr unsigned char kMagic[4] = {'A', 'T', 'K', 'V'};
constexpr unsigned kVersion = 1;
constexpr size_t kHeaderBytes = 21;
constexpr uint64_t kMaxValues = 1ull << 34;      // dataset.cpp:98 "dataset too large"
constexpr size_t kChunkValues = size_t(1) << 22;  // 16 MiB staging chunks

void put_u64_le(unsigned char* out, uint64_t v) {
  for (int i = 0; i < 8; ++i) out[i] = static_cast<unsigned char>(v >> (8 * i));
}
uint64_t get_u64_le(const unsigned char* in) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(in[i]) << (8 * i);
  return v;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

struct Pinned {
  void* p = nullptr;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

// dataset.cpp:84-101: header read and checks, in the reference's order.
void read_header(FILE* f, uint64_t* rows, uint64_t* dims) {
  unsigned char h[kHeaderBytes];
  if (std::fread(h, 1, kHeaderBytes, f) != kHeaderBytes)
    throw FormatError("dataset truncated: header incomplete");
  if (std::memcmp(h, kMagic, 4) != 0) throw FormatError("bad dataset magic");
  if (h[4] != kVersion) throw FormatError("unsupported dataset version " + std::to_string(h[4]));
  const uint64_t r = get_u64_le(h + 5), d = get_u64_le(h + 13);
  if (d != 0 && r > UINT64_MAX / d) throw FormatError("dataset shape overflows");
  if (r * d > kMaxValues) throw FormatError("dataset too large");
  *rows = r;
  *dims = d;
}

// dataset.cpp:37-41 (VectorDataset::validate), shape half
void check_shape(uint64_t rows, uint64_t dims) {
  if (dims != 0 && rows > UINT64_MAX / dims) throw FormatError("dataset shape overflows");
}

void open_read(File& f, const char* path) {
  f.f = path ? std::fopen(path, "rb") : nullptr;
  if (!f.f) throw FormatError(std::string("cannot open for read: ") + (path ? path : ""));
}
void open_write(File& f, const char* path) {
  f.f = path ? std::fopen(path, "wb") : nullptr;
  if (!f.f) throw FormatError(std::string("cannot open for write: ") + (path ? path : ""));
}

void write_header(FILE* f, uint64_t rows, uint64_t dims) {
  unsigned char h[kHeaderBytes];
  std::memcpy(h, kMagic, 4);
  h[4] = static_cast<unsigned char>(kVersion);
  put_u64_le(h + 5, rows);
  put_u64_le(h + 13, dims);
  if (std::fwrite(h, 1, kHeaderBytes, f) != kHeaderBytes) throw FormatError("dataset write failed");
}

bool host_has_nan(const float* x, uint64_t count) {
  const uint32_t* b = reinterpret_cast<const uint32_t*>(x);
  uint32_t any = 0;
  for (uint64_t i = 0; i < count; ++i) any |= (b[i] & 0x7fffffffu) > 0x7f800000u;
  return any != 0;
}

// HBM-bound NaN scan: 16-byte loads when the buffer is 16-byte aligned (scalar
// loads otherwise, e.g. a row-offset view), grid-stride, one atomic per warp that
// sees a NaN.
__global__ void __launch_bounds__(256) nan_scan_kernel(const float* __restrict__ x, uint64_t count,
                                                       bool vec, uint32_t* __restrict__ flag) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t nvec = vec ? count / 4 : 0;
  const uint4* v = reinterpret_cast<const uint4*>(x);
  bool nan = false;
  for (uint64_t i = tid; i < nvec; i += nthreads) {
    const uint4 w = __ldg(v + i);
    nan |= ((w.x & 0x7fffffffu) > 0x7f800000u) | ((w.y & 0x7fffffffu) > 0x7f800000u) |
           ((w.z & 0x7fffffffu) > 0x7f800000u) | ((w.w & 0x7fffffffu) > 0x7f800000u);
  }
  for (uint64_t i = nvec * 4 + tid; i < count; i += nthreads)
    nan |= (__float_as_uint(__ldg(x + i)) & 0x7fffffffu) > 0x7f800000u;
  if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

void launch_nan_scan(const float* d, uint64_t count, uint32_t* flag, cudaStream_t s) {
  if (count == 0) return;
  const bool vec = reinterpret_cast<uintptr_t>(d) % 16 == 0;
  const uint64_t want = ((vec ? count / 4 : count) + 255) / 256;
  const uint64_t cap = uint64_t(sm_count()) * 8;
  const unsigned grid = static_cast<unsigned>(want < 1 ? 1 : (want > cap ? cap : want));
  nan_scan_kernel<<<grid, 256, 0, s>>>(d, count, vec, flag);
  check_launch();
}

}  // namespace
}  // namespace atkg

using namespace atkg;

namespace {
// DatasetFormatError (dataset.hpp:14-16) gets its own status code, ATKG_EFORMAT;
// every other failure goes through guarded().
template <class F>
int run_io(F&& f) {
  std::string fmt;
  const int rc = guarded([&] {
    try {
      f();
    } catch (const FormatError& e) {
      fmt = e.what();
    }
  });
  if (rc == ATKG_OK && !fmt.empty()) {
    set_last_error(fmt);
    return ATKG_EFORMAT;
  }
  return rc;
}
}  // namespace

extern "C" {

int atkg_dataset_read_header(const char* path, uint64_t* rows, uint64_t* dims) {
  return run_io([&] {
    if (!rows || !dims) throw Inval("rows/dims out-pointers must not be null");
    File f;
    open_read(f, path);
    read_header(f.f, rows, dims);
  });
}

int atkg_dataset_read_file(const char* path, float* out, uint64_t capacity, uint64_t* rows,
                           uint64_t* dims) {
  return run_io([&] {
    if (!rows || !dims) throw Inval("rows/dims out-pointers must not be null");
    File f;
    open_read(f, path);
    uint64_t r, d;
    read_header(f.f, &r, &d);
    const uint64_t total = r * d;
    if (total > capacity) throw Inval("output buffer too small for the dataset payload");
    if (total && !out) throw Inval("output buffer must not be null");
    // dataset.cpp:104-121: chunked read, truncation reported as soon as a chunk is short
    for (uint64_t i = 0; i < total;) {
      const uint64_t count = std::min<uint64_t>(kChunkValues, total - i);
      if (std::fread(out + i, 4, count, f.f) != count)
        throw FormatError("dataset truncated: payload incomplete");
      i += count;
    }
    if (host_has_nan(out, total)) throw FormatError("dataset payload contains NaN");
    *rows = r;
    *dims = d;
  });
}

int atkg_dataset_write_file(const char* path, const float* data, uint64_t rows, uint64_t dims) {
  return run_io([&] {
    File f;
    open_write(f, path);  // dataset.cpp:75-80 opens before validating
    check_shape(rows, dims);
    const uint64_t total = rows * dims;
    if (total && !data) throw Inval("input buffer must not be null");
    if (host_has_nan(data, total)) throw FormatError("dataset payload contains NaN");
    write_header(f.f, rows, dims);
    if (total && std::fwrite(data, 4, total, f.f) != total) throw FormatError("dataset write failed");
    if (std::fflush(f.f) != 0) throw FormatError("dataset write failed");
  });
}

int atkg_dataset_read_file_device(const char* path, float* d_out, uint64_t capacity, uint64_t* rows,
                                  uint64_t* dims, void* stream) {
  return run_io([&] {
    if (!rows || !dims) throw Inval("rows/dims out-pointers must not be null");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    File f;
    open_read(f, path);
    uint64_t r, d;
    read_header(f.f, &r, &d);
    const uint64_t total = r * d;
    if (total > capacity) throw Inval("output buffer too small for the dataset payload");
    if (total && !d_out) throw Inval("output buffer must not be null");
    uint32_t* d_flag = nullptr;
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_flag), sizeof(uint32_t), s));
    std::unique_ptr<uint32_t, void (*)(uint32_t*)> flag_guard(d_flag, [](uint32_t* p) { cudaFree(p); });
    CUDA_OK(cudaMemsetAsync(d_flag, 0, sizeof(uint32_t), s));
    const uint64_t chunk = std::min<uint64_t>(kChunkValues, total ? total : 1);
    Pinned buf[2];
    cudaEvent_t done[2] = {nullptr, nullptr};
    std::unique_ptr<cudaEvent_t, void (*)(cudaEvent_t*)> ev_guard(done, [](cudaEvent_t* e) {
      for (int j = 0; j < 2; ++j)
        if (e[j]) cudaEventDestroy(e[j]);
    });
    for (int j = 0; j < 2; ++j) {
      CUDA_OK(cudaHostAlloc(&buf[j].p, chunk * 4, cudaHostAllocDefault));
      CUDA_OK(cudaEventCreateWithFlags(&done[j], cudaEventDisableTiming));
    }
    // Double buffer: the file read of chunk c+1 overlaps the H2D copy of chunk c.
    uint64_t c = 0;
    for (uint64_t i = 0; i < total; ++c) {
      const uint64_t count = std::min<uint64_t>(chunk, total - i);
      float* h = static_cast<float*>(buf[c & 1].p);
      CUDA_OK(cudaEventSynchronize(done[c & 1]));  // previous copy out of this buffer finished
      if (std::fread(h, 4, count, f.f) != count) {
        cudaStreamSynchronize(s);
        throw FormatError("dataset truncated: payload incomplete");
      }
      CUDA_OK(cudaMemcpyAsync(d_out + i, h, count * 4, cudaMemcpyHostToDevice, s));
      CUDA_OK(cudaEventRecord(done[c & 1], s));
      i += count;
    }
    launch_nan_scan(d_out, total, d_flag, s);
    uint32_t flag = 0;
    CUDA_OK(cudaMemcpyAsync(&flag, d_flag, sizeof flag, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (flag) throw FormatError("dataset payload contains NaN");
    *rows = r;
    *dims = d;
  });
}

int atkg_dataset_write_file_device(const char* path, const float* d_in, uint64_t rows, uint64_t dims,
                                   void* stream) {
  return run_io([&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    File f;
    open_write(f, path);
    check_shape(rows, dims);
    const uint64_t total = rows * dims;
    if (total && !d_in) throw Inval("input buffer must not be null");
    uint32_t* d_flag = nullptr;
    CUDA_OK(cudaMallocAsync(reinterpret_cast<void**>(&d_flag), sizeof(uint32_t), s));
    std::unique_ptr<uint32_t, void (*)(uint32_t*)> flag_guard(d_flag, [](uint32_t* p) { cudaFree(p); });
    CUDA_OK(cudaMemsetAsync(d_flag, 0, sizeof(uint32_t), s));
    launch_nan_scan(d_in, total, d_flag, s);
    uint32_t flag = 0;
    CUDA_OK(cudaMemcpyAsync(&flag, d_flag, sizeof flag, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (flag) throw FormatError("dataset payload contains NaN");
    write_header(f.f, rows, dims);
    const uint64_t chunk = std::min<uint64_t>(kChunkValues, total ? total : 1);
    Pinned buf[2];
    cudaEvent_t done[2] = {nullptr, nullptr};
    std::unique_ptr<cudaEvent_t, void (*)(cudaEvent_t*)> ev_guard(done, [](cudaEvent_t* e) {
      for (int j = 0; j < 2; ++j)
        if (e[j]) cudaEventDestroy(e[j]);
    });
    for (int j = 0; j < 2; ++j) {
      CUDA_OK(cudaHostAlloc(&buf[j].p, chunk * 4, cudaHostAllocDefault));
      CUDA_OK(cudaEventCreateWithFlags(&done[j], cudaEventDisableTiming));
    }
    // D2H of chunk c+1 is queued before chunk c is written to the file.
    const uint64_t nchunks = (total + chunk - 1) / chunk;
    auto issue = [&](uint64_t c) {
      const uint64_t off = c * chunk, count = std::min<uint64_t>(chunk, total - off);
      CUDA_OK(cudaMemcpyAsync(buf[c & 1].p, d_in + off, count * 4, cudaMemcpyDeviceToHost, s));
      CUDA_OK(cudaEventRecord(done[c & 1], s));
    };
    if (nchunks) issue(0);
    for (uint64_t c = 0; c < nchunks; ++c) {
      CUDA_OK(cudaEventSynchronize(done[c & 1]));
      if (c + 1 < nchunks) issue(c + 1);
      const uint64_t count = std::min<uint64_t>(chunk, total - c * chunk);
      if (std::fwrite(buf[c & 1].p, 4, count, f.f) != count) {
        cudaStreamSynchronize(s);
        throw FormatError("dataset write failed");
      }
    }
    if (std::fflush(f.f) != 0) throw FormatError("dataset write failed");
  });
}

}  // extern "C"
