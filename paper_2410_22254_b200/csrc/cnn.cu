// MNIST CNN pack (placeholder until the conv kernels land).
#include "pack.cuh"

namespace tlk {

int cnn_setup(Pack& p) {
  (void)p;
  return fail(TLK_EINVAL, "cnn model not built yet");
}
int cnn_enqueue_step(Pack& p, cudaStream_t st) {
  (void)p;
  (void)st;
  return fail(TLK_EINVAL, "cnn model not built yet");
}

}  // namespace tlk
