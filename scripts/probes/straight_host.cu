// Host for gen_straight_probe.py cubins: loads a cubin with the driver API and
// reports FP32 FMA throughput (useful FMAs = 32 per case per lane).
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { CUresult e_ = (x); if (e_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(e_, &s); printf("%s: %s\n", #x, s); exit(1);} } while (0)
int main(int argc, char** argv) {
  // argv: cubin M mode ctas_per_sm
  const char* path = argv[1]; int M = atoi(argv[2]); unsigned mode = atoi(argv[3]); int cps = argc > 4 ? atoi(argv[4]) : 1;
  CK(cuInit(0)); CUdevice dev; CK(cuDeviceGet(&dev, 0)); CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CUmodule mod; CK(cuModuleLoad(&mod, path)); CUfunction f; CK(cuModuleGetFunction(&f, mod, "probe"));
  int ctas = 148 * cps; CUdeviceptr out; CK(cuMemAlloc(&out, ctas * 256 * 4));
  unsigned reps = 4;
  void* args[] = {&out, &reps, &mode};
  CK(cuLaunchKernel(f, ctas, 1, 1, 256, 1, 1, 0, 0, args, 0)); CK(cuCtxSynchronize());
  reps = (unsigned)(400000 / M); if (reps < 2) reps = 2;
  CUevent a, b; CK(cuEventCreate(&a, 0)); CK(cuEventCreate(&b, 0));
  CK(cuEventRecord(a, 0)); CK(cuLaunchKernel(f, ctas, 1, 1, 256, 1, 1, 0, 0, args, 0)); CK(cuEventRecord(b, 0));
  CK(cuEventSynchronize(b)); float ms; CK(cuEventElapsedTime(&ms, a, b));
  double fl = 2.0 * 32 * M * 256.0 * ctas * reps;
  printf("%s M=%d mode=%u ctas=%d: %.3f ms  %.1f TFLOP/s  (%.1f%% of 74.4)\n", path, M, mode, ctas, ms, fl / ms / 1e9, fl / ms / 1e9 / 74.4 * 100);
  return 0;
}
