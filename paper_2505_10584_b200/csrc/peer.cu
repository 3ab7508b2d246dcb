// Peer memory over NVLink / NVSwitch for the fused Ulysses exchange.
//
// The paper's multi-xPU path swaps sequence shards for head shards around
// attention (the reference only costs it, comm.py:65-96).
// Instead of an NCCL all-to-all between a packing kernel and attention, the
// producing kernels store straight into the consumer rank's buffer:
//   * the QKV GEMM epilogue TMA-stores each head group into the owning
//     rank's attention-input buffer (aqb_gemm_qknorm_rope_scatter);
//   * the attention epilogue stores each output row into the owning rank's
//     O buffer (aqb_attention_fwd_scatter).
// These buffers are plain cudaMalloc allocations shared with CUDA IPC; the
// only synchronisation left is aqb_peer_barrier — one tiny kernel in which
// every rank publishes an epoch number into each peer's signal slots
// (st.release.sys) and spins (ld.acquire.sys) until all peers published
// theirs.  It optionally carries a few floats per rank and reduces them in
// rank order, identically on every rank (the diffusion-cache rel-L1 sums).
#include <cstring>

#include "host.cuh"

namespace aqb {
namespace peer {

constexpr int kMaxRanks = 8;
constexpr int kMaxPay = 4;

// Signal region (one per rank, in peer memory; AQB_PEER_SIGNAL_BYTES).
struct Signal {
  uint32_t flag[kMaxRanks];                // flag[src] = last epoch rank src reached
  uint32_t pad[8];
  float pay[2][kMaxRanks][kMaxPay];        // payload, double-buffered by epoch parity
};
static_assert(sizeof(Signal) <= AQB_PEER_SIGNAL_BYTES, "signal region");

struct BarrierArgs {
  Signal* sig[kMaxRanks];
  int rank, nranks, npay;
  uint32_t* epoch;
  const float* payload;
  float* pay_out;
  int32_t* status;
  const int32_t* run_flag;
  int32_t run_if;
  long long timeout_cycles;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(32) barrier_kernel(BarrierArgs a) {
  // PDL: launched while the producer drains; its writes (incl. remote TMA stores) are
  // complete and visible from here.  Triggering at once lets the consumer's prologue
  // overlap the spin (the consumer's own griddepcontrol.wait still waits for this kernel).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.run_flag != nullptr && *a.run_flag != a.run_if) return;
  const int t = threadIdx.x;
  const uint32_t e = *a.epoch + 1;
  const int par = e & 1;
  // every prior write of this rank (previous kernels, incl. remote TMA stores — complete
  // before those kernels exited, and visible here after griddepcontrol.wait) is ordered
  // before the signal: an acq_rel system fence (cumulative), then a release store, which
  // also orders this thread's payload writes
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (t < a.nranks) {
    Signal* dst = a.sig[t];
    for (int i = 0; i < a.npay; ++i) dst->pay[par][a.rank][i] = a.payload[i];
    st_release_sys(&dst->flag[a.rank], e);
  }
  if (t < a.nranks) {
    const uint32_t* f = &a.sig[a.rank]->flag[t];
    const long long t0 = clock64();
    while (static_cast<int32_t>(ld_acquire_sys(f) - e) < 0) {
      if (clock64() - t0 > a.timeout_cycles) {  // a peer never arrived: report, never hang the GPU
        if (a.status) atomicExch(a.status, 1);
        break;
      }
    }
  }
  // each thread reads the payload of the rank whose flag it acquired; the sum
  // runs in rank order (shuffles), so every rank gets bit-identical results
  for (int i = 0; i < a.npay; ++i) {
    const float v = t < a.nranks ? *reinterpret_cast<volatile const float*>(&a.sig[a.rank]->pay[par][t][i]) : 0.f;
    float s = 0.f;
    for (int r = 0; r < a.nranks; ++r) s += __shfl_sync(0xffffffffu, v, r);
    if (t == 0) a.pay_out[i] = s;
  }
  __syncwarp();
  if (t == 0) {
    *a.epoch = e;
  }
}

}  // namespace peer
}  // namespace aqb

extern "C" {

int aqb_peer_alloc(int64_t bytes, void** ptr, void* ipc_handle) {
  using namespace aqb;
  AQB_CHECK_ARG(bytes > 0 && ptr && ipc_handle, "peer_alloc: bad arguments");
  void* p = nullptr;
  AQB_CUDA_TRY(cudaMalloc(&p, static_cast<size_t>(bytes)));
  AQB_CUDA_TRY(cudaMemset(p, 0, static_cast<size_t>(bytes)));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return set_error(AQB_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == AQB_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(ipc_handle, &h, sizeof(h));
  *ptr = p;
  return AQB_OK;
}

int aqb_peer_open(const void* ipc_handle, void** ptr) {
  using namespace aqb;
  AQB_CHECK_ARG(ipc_handle && ptr, "peer_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  AQB_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return AQB_OK;
}

int aqb_peer_close(void* ptr) {
  using namespace aqb;
  AQB_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return AQB_OK;
}

int aqb_peer_free(void* ptr) {
  using namespace aqb;
  AQB_CUDA_TRY(cudaFree(ptr));
  return AQB_OK;
}

int aqb_peer_can_access(int32_t device, int32_t peer_device) {
  int ok = 0;
  if (cudaDeviceCanAccessPeer(&ok, device, peer_device) != cudaSuccess) return 0;
  return ok;
}

int aqb_peer_barrier(void* const* peer_signal, int32_t rank, int32_t nranks, uint32_t* epoch, const float* payload,
                     int32_t npay, float* pay_out, int32_t* status, const int32_t* run_flag, int32_t run_if,
                     void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(peer_signal && epoch, "peer_barrier: null pointer");
  AQB_CHECK_ARG(nranks >= 1 && nranks <= peer::kMaxRanks && rank >= 0 && rank < nranks, "peer_barrier: rank %d/%d",
                rank, nranks);
  AQB_CHECK_ARG(npay >= 0 && npay <= peer::kMaxPay && (npay == 0 || (payload && pay_out)), "peer_barrier: payload");
  peer::BarrierArgs a{};
  for (int r = 0; r < nranks; ++r) {
    AQB_CHECK_ARG(peer_signal[r] != nullptr, "peer_barrier: signal[%d] is null", r);
    a.sig[r] = reinterpret_cast<peer::Signal*>(peer_signal[r]);
  }
  a.rank = rank, a.nranks = nranks, a.npay = npay, a.epoch = epoch;
  a.payload = payload, a.pay_out = pay_out, a.status = status;
  a.run_flag = run_flag, a.run_if = run_if;
  a.timeout_cycles = 20ll * 1000 * 1000 * 1000;  // ~10 s at 2 GHz
  AQB_CUDA_TRY(launch_pdl(peer::barrier_kernel, dim3(1), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), a));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

}  // extern "C"
