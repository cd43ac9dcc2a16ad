// GPU unit test of LL32's per-line completeness check (paper_2506_20252_b200/csrc/transport.cuh,
// ld_line32 / line_hash). A 32-byte line is two 16-byte sectors {w0..w3} {w4..w6, check}; a torn
// arrival shows one sector of the new store and one of the old line. The receiver must not
// accept such a line, nor a stale line of another step, nor a zeroed line; it must accept the
// line once both sectors are the new store's. Exit code 0 = every case behaved.
#include <cstdio>
#include <cstring>

#include "../../paper_2506_20252_b200/csrc/transport.cuh"

using namespace pat;

__global__ void poll_kernel(const char* line, uint32_t flag, uint64_t timeout_ns, int* err, int* ok, uint32_t* words) {
  Waiter w{timeout_ns, err, false, true};
  const Line32 v = ld_line32(line, flag, w);
  *ok = w.aborted ? 0 : 1;
  for (int k = 0; k < 8; ++k) words[k] = v.w[k];
}

static int poll(char* dline, const Line32& host, uint32_t flag, int* d_ok, int* d_err, uint32_t* d_words,
                uint32_t* got) {
  cudaMemcpy(dline, &host, 32, cudaMemcpyHostToDevice);
  cudaMemset(d_err, 0, sizeof(int));
  poll_kernel<<<1, 1>>>(dline, flag, 2000000ull /* 2 ms */, d_err, d_ok, d_words);
  int ok = -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  cudaMemcpy(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(got, d_words, 32, cudaMemcpyDeviceToHost);
  return ok;
}

int main() {
  char* dline;
  int *d_ok, *d_err;
  uint32_t* d_words;
  cudaMalloc(&dline, 64);
  cudaMalloc(&d_ok, sizeof(int));
  cudaMalloc(&d_err, sizeof(int));
  cudaMalloc(&d_words, 32);
  uint32_t got[8];
  int fails = 0;
  const uint32_t step_flag = 1001, old_flag = 1001 - 4;  // this step, the step that last used the slot
  for (int trial = 0; trial < 64; ++trial) {
    Line32 nw{}, od{};
    for (int k = 0; k < 7; ++k) {
      nw.w[k] = 0x12345u * (trial + 1) + 977u * k + (trial & 1 ? 0 : k * 0x01010101u);
      od.w[k] = nw.w[k] ^ (1u << ((trial + k) % 32));  // old data: one bit away per word
    }
    if (trial % 4 == 3) od.w[trial % 7] = nw.w[trial % 7] + 1;  // a single word differs by one
    nw.w[7] = step_flag ^ line_hash(nw);
    od.w[7] = old_flag ^ line_hash(od);
    Line32 torn_a = nw, torn_b = nw;
    for (int k = 0; k < 4; ++k) torn_a.w[k] = od.w[k];       // check sector new, data sector old
    for (int k = 4; k < 8; ++k) torn_b.w[k] = od.w[k];       // data sector new, check sector old
    const Line32* rejected[3] = {&torn_a, &torn_b, &od};
    for (int i = 0; i < 3; ++i) {
      const int ok = poll(dline, *rejected[i], step_flag, d_ok, d_err, d_words, got);
      if (ok != 0) {
        std::printf("trial %d case %d: accepted a torn/stale line (ok=%d)\n", trial, i, ok);
        ++fails;
      }
    }
    const int ok = poll(dline, nw, step_flag, d_ok, d_err, d_words, got);
    if (ok != 1 || std::memcmp(got, nw.w, 32) != 0) {
      std::printf("trial %d: complete line not accepted (ok=%d)\n", trial, ok);
      ++fails;
    }
  }
  // a zeroed line (fresh pool) is never complete for a nonzero step value
  Line32 zero{};
  if (poll(dline, zero, step_flag, d_ok, d_err, d_words, got) != 0) {
    std::printf("zero line accepted\n");
    ++fails;
  }
  // the epoch re-stamp {0 x 7, V}: complete for V only
  Line32 stamp{};
  stamp.w[7] = step_flag - 0x40000000u;
  if (poll(dline, stamp, step_flag, d_ok, d_err, d_words, got) != 0 ||
      poll(dline, stamp, step_flag - 0x40000000u, d_ok, d_err, d_words, got) != 1) {
    std::printf("epoch stamp misjudged\n");
    ++fails;
  }
  std::printf("%s: ll32 tear cases, %d failures\n", fails ? "FAIL" : "ok", fails);
  return fails ? 1 : 0;
}
