// abi.cu -- status / error plumbing and descriptor validation of the C ABI.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace cacto {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CACTO_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return CACTO_OK;
}

bool ensure_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(kernel);
  if (it != done.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  done[kernel] = bytes;
  return true;
}

}  // namespace cacto

using namespace cacto;

int validate_mlp(const cacto_mlp_t* m, const char* who) {
  if (!m) return set_error(CACTO_EVALUE, "%s: null network", who);
  if (m->dtype != CACTO_F32 && m->dtype != CACTO_F64) return set_error(CACTO_EVALUE, "%s: bad dtype", who);
  if (m->n_layers < 1 || m->n_layers > CACTO_MAX_LAYERS)
    return set_error(CACTO_EUNSUPPORTED, "%s: %d layers not supported", who, m->n_layers);
  if (m->sizes[0] < 1 || m->sizes[0] > CACTO_MAX_IN)
    return set_error(CACTO_EUNSUPPORTED, "%s: input width %d not supported", who, m->sizes[0]);
  int out = m->sizes[m->n_layers];
  if (out < 1 || out > CACTO_MAX_OUT) return set_error(CACTO_EUNSUPPORTED, "%s: output width %d not supported", who, out);
  if (m->n_layers > 1 && m->hp != 32 && m->hp != 64 && (m->hp % 32 || m->hp > CACTO_MAX_HIDDEN))
    return set_error(CACTO_EUNSUPPORTED, "%s: padded hidden width %d not supported", who, m->hp);
  if (m->n_layers > 1 && m->hp > 64 && m->dtype != CACTO_F32)
    return set_error(CACTO_EUNSUPPORTED, "%s: padded hidden width %d > 64 runs in fp32 only", who, m->hp);
  for (int i = 1; i < m->n_layers; ++i)
    if (m->sizes[i] < 1 || m->sizes[i] > m->hp)
      return set_error(CACTO_EVALUE, "%s: hidden width %d exceeds padded width %d", who, m->sizes[i], m->hp);
  if (m->activation != CACTO_ACT_ELU && m->activation != CACTO_ACT_TANH)
    return set_error(CACTO_EVALUE, "%s: unknown activation", who);
  if (m->head < CACTO_HEAD_LINEAR || m->head > CACTO_HEAD_STD) return set_error(CACTO_EVALUE, "%s: unknown head", who);
  if (!m->params) return set_error(CACTO_EVALUE, "%s: null parameter buffer", who);
  return CACTO_OK;
}

extern "C" int cacto_abi_version(void) { return CACTO_ABI_VERSION; }
extern "C" const char* cacto_last_error(void) { return g_err; }
extern "C" int32_t cacto_padded_in(int32_t in_dim) { return padded_in(in_dim); }
extern "C" int64_t cacto_mlp_param_count(const cacto_mlp_t* mlp) {
  if (!mlp || mlp->n_layers < 1 || mlp->n_layers > CACTO_MAX_LAYERS) return -1;
  cacto_mlp_t m = *mlp;
  if (m.n_layers == 1) m.hp = 0;
  return layer_offsets(shape_of(m)).total;
}
