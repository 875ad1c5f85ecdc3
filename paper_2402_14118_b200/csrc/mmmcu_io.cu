// mmmcu_io.cu — MMMB matrix files straight into / out of device memory (C ABI, include/mmmcu.h).
//
// The reference's interchange format (/root/reference/proj/include/mmm/matrix_io.hpp:11-13,
// src/matrix_io.cpp): little-endian "MMMB" | u32 version = 1 | u32 dtype (0 = f32, 1 = f64) |
// u64 rows | u64 cols | rows*cols elements, row-major, no padding.  Loading rebuilds the
// Matrix padding on the device (ld columns per row, columns [cols, ld) zero, matrix.hpp:82),
// streaming the payload through a pinned staging buffer in row blocks so that large operands
// (configs[3]'s 2.25 GiB B) never need a host copy of the whole matrix.  Error classes follow
// matrix_io.hpp:15-29: bad magic / unsupported version / unknown dtype / truncated / I/O.
#include "../../include/mmmcu.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

namespace {

thread_local std::string g_io_err;

mmmcu_status io_fail(mmmcu_status s, const std::string& m) {
  g_io_err = m;
  return s;
}

struct FileCloser {
  void operator()(std::FILE* f) const {
    if (f) std::fclose(f);
  }
};
using File = std::unique_ptr<std::FILE, FileCloser>;

struct PinnedBuf {
  void* p = nullptr;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

constexpr size_t kStageBytes = size_t(64) << 20;  // pinned staging per block of rows

mmmcu_status read_header(std::FILE* f, const char* path, uint32_t* dtype, uint64_t* rows, uint64_t* cols) {
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4) return io_fail(MMMCU_ERR_FILE_TRUNCATED, std::string("truncated header in ") + path);
  if (std::memcmp(magic, "MMMB", 4) != 0) return io_fail(MMMCU_ERR_FILE_FORMAT, std::string("bad magic in ") + path);
  uint32_t version = 0;
  if (std::fread(&version, 4, 1, f) != 1) return io_fail(MMMCU_ERR_FILE_TRUNCATED, std::string("truncated header in ") + path);
  if (version != 1) return io_fail(MMMCU_ERR_FILE_FORMAT, std::string("unsupported format version in ") + path);
  if (std::fread(dtype, 4, 1, f) != 1) return io_fail(MMMCU_ERR_FILE_TRUNCATED, std::string("truncated header in ") + path);
  if (*dtype > 1) return io_fail(MMMCU_ERR_FILE_FORMAT, std::string("unknown dtype code in ") + path);
  if (std::fread(rows, 8, 1, f) != 1 || std::fread(cols, 8, 1, f) != 1)
    return io_fail(MMMCU_ERR_FILE_TRUNCATED, std::string("truncated header in ") + path);
  if (*rows == 0 || *cols == 0) return io_fail(MMMCU_ERR_FILE_FORMAT, std::string("zero dimension in ") + path);
  return MMMCU_OK;
}

}  // namespace

extern "C" {

const char* mmmcu_io_last_error(void) { return g_io_err.c_str(); }

mmmcu_status mmmcu_mmmb_peek(const char* path, int32_t* dtype, int64_t* rows, int64_t* cols) {
  if (!path || !dtype || !rows || !cols) return io_fail(MMMCU_ERR_INVALID_ARG, "null argument");
  File f(std::fopen(path, "rb"));
  if (!f) return io_fail(MMMCU_ERR_FILE_IO, std::string("cannot open ") + path);
  uint32_t dt = 0;
  uint64_t r = 0, c = 0;
  const mmmcu_status s = read_header(f.get(), path, &dt, &r, &c);
  if (s != MMMCU_OK) return s;
  *dtype = (int32_t)dt;
  *rows = (int64_t)r;
  *cols = (int64_t)c;
  return MMMCU_OK;
}

mmmcu_status mmmcu_mmmb_load(const char* path, float* dev, int64_t ld, int64_t max_rows, void* stream, int64_t* rows,
                             int64_t* cols) {
  if (!path || !dev || !rows || !cols) return io_fail(MMMCU_ERR_INVALID_ARG, "null argument");
  File f(std::fopen(path, "rb"));
  if (!f) return io_fail(MMMCU_ERR_FILE_IO, std::string("cannot open ") + path);
  uint32_t dt = 0;
  uint64_t r = 0, c = 0;
  mmmcu_status s = read_header(f.get(), path, &dt, &r, &c);
  if (s != MMMCU_OK) return s;
  if (dt != 0) return io_fail(MMMCU_ERR_UNSUPPORTED, std::string(path) + " holds f64: the GPU path is f32 only");
  *rows = (int64_t)r;
  *cols = (int64_t)c;
  if ((int64_t)c > ld || (int64_t)r > max_rows)
    return io_fail(MMMCU_ERR_DIM_MISMATCH, "device buffer too small for " + std::to_string(r) + " x " + std::to_string(c));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // zero padding columns (and nothing else is required: every logical element is written)
  if (ld > (int64_t)c) {
    cudaError_t e = cudaMemset2DAsync(dev + c, sizeof(float) * ld, 0, sizeof(float) * (ld - c), r, st);
    if (e != cudaSuccess) return io_fail(MMMCU_ERR_CUDA, cudaGetErrorString(e));
  }
  const size_t row_bytes = sizeof(float) * c;
  const size_t block_rows = std::max<size_t>(1, kStageBytes / row_bytes);
  PinnedBuf stage[2];
  for (auto& b : stage)
    if (cudaMallocHost(&b.p, block_rows * row_bytes) != cudaSuccess) return io_fail(MMMCU_ERR_CUDA, "pinned staging");
  cudaEvent_t done[2];
  cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming);
  bool used[2] = {false, false};
  for (uint64_t r0 = 0, blk = 0; r0 < r; r0 += block_rows, ++blk) {
    const int b = (int)(blk & 1);
    if (used[b]) cudaEventSynchronize(done[b]);  // the copy from this staging buffer finished
    const size_t nr = std::min<uint64_t>(block_rows, r - r0);
    if (std::fread(stage[b].p, 1, nr * row_bytes, f.get()) != nr * row_bytes) {
      cudaStreamSynchronize(st);
      cudaEventDestroy(done[0]);
      cudaEventDestroy(done[1]);
      return io_fail(MMMCU_ERR_FILE_TRUNCATED, std::string("truncated payload in ") + path);
    }
    cudaError_t e = cudaMemcpy2DAsync(dev + r0 * ld, sizeof(float) * ld, stage[b].p, row_bytes, row_bytes, nr,
                                      cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventRecord(done[b], st);
    if (e != cudaSuccess) {
      cudaStreamSynchronize(st);
      cudaEventDestroy(done[0]);
      cudaEventDestroy(done[1]);
      return io_fail(MMMCU_ERR_CUDA, cudaGetErrorString(e));
    }
    used[b] = true;
  }
  const cudaError_t e = cudaStreamSynchronize(st);  // staging is freed on return
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
  if (e != cudaSuccess) return io_fail(MMMCU_ERR_CUDA, cudaGetErrorString(e));
  return MMMCU_OK;
}

mmmcu_status mmmcu_mmmb_save(const char* path, const float* dev, int64_t rows, int64_t cols, int64_t ld, void* stream) {
  if (!path || !dev || rows <= 0 || cols <= 0 || ld < cols) return io_fail(MMMCU_ERR_INVALID_ARG, "bad arguments");
  File f(std::fopen(path, "wb"));
  if (!f) return io_fail(MMMCU_ERR_FILE_IO, std::string("cannot open ") + path);
  const uint32_t version = 1, dtype = 0;
  const uint64_t r = (uint64_t)rows, c = (uint64_t)cols;
  if (std::fwrite("MMMB", 1, 4, f.get()) != 4 || std::fwrite(&version, 4, 1, f.get()) != 1 ||
      std::fwrite(&dtype, 4, 1, f.get()) != 1 || std::fwrite(&r, 8, 1, f.get()) != 1 || std::fwrite(&c, 8, 1, f.get()) != 1)
    return io_fail(MMMCU_ERR_FILE_IO, std::string("short write to ") + path);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t row_bytes = sizeof(float) * c;
  const size_t block_rows = std::max<size_t>(1, kStageBytes / row_bytes);
  PinnedBuf stage;
  if (cudaMallocHost(&stage.p, block_rows * row_bytes) != cudaSuccess) return io_fail(MMMCU_ERR_CUDA, "pinned staging");
  for (uint64_t r0 = 0; r0 < r; r0 += block_rows) {
    const size_t nr = std::min<uint64_t>(block_rows, r - r0);
    cudaError_t e = cudaMemcpy2DAsync(stage.p, row_bytes, dev + r0 * ld, sizeof(float) * ld, row_bytes, nr,
                                      cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return io_fail(MMMCU_ERR_CUDA, cudaGetErrorString(e));
    if (std::fwrite(stage.p, 1, nr * row_bytes, f.get()) != nr * row_bytes)
      return io_fail(MMMCU_ERR_FILE_IO, std::string("short write to ") + path);
  }
  if (std::fflush(f.get()) != 0) return io_fail(MMMCU_ERR_FILE_IO, std::string("flush failed for ") + path);
  return MMMCU_OK;
}

}  // extern "C"
