// transport_kernels.cu — instantiates K1 for one arithmetic type.
// Compiled twice by the build: once with -DVMC_REAL=float (FMA contraction on,
// the product path) and once with -DVMC_REAL=double --fmad=false (parity mode;
// no contraction, like the reference built with -ffp-contract=off).
#include "transport.cuh"
#include "flight.cuh"

#ifndef VMC_REAL
#define VMC_REAL float
#endif

namespace vmc {

// Occupancy: every FP32 variant is capped at 64 registers (4 CTAs = 32 warps per
// SM). The plain kernel also fits 48 registers without spills (5 CTAs), which
// measured 1-2 % slower: the loop is issue-bound, not latency-bound. FP64
// (parity mode) is unconstrained.
#ifndef VMC_MIN_BLOCKS
#if VMC_REAL_IS_FLOAT
#define VMC_MIN_BLOCKS_PLAIN 4
#define VMC_MIN_BLOCKS_RICH 4
#else
#define VMC_MIN_BLOCKS_PLAIN 1
#define VMC_MIN_BLOCKS_RICH 1
#endif
#else
#define VMC_MIN_BLOCKS_PLAIN VMC_MIN_BLOCKS
#define VMC_MIN_BLOCKS_RICH VMC_MIN_BLOCKS
#endif
template <typename Real, bool G, bool D, bool T, bool U = false>
__global__ void __launch_bounds__(kBlock, (G || D || T) ? VMC_MIN_BLOCKS_RICH : VMC_MIN_BLOCKS_PLAIN)
    k_transport(const __grid_constant__ KernelArgs A) {
  transport_body<Real, G, D, T, U>(A);
}

#define VMC_CAT2(a, b) a##b
#define VMC_CAT(a, b) VMC_CAT2(a, b)

// Returns the kernel for (gates, detectors, trace, single-label volume); host
// code launches it with cudaLaunchKernel and sizes the persistent grid by
// occupancy. The single-label specialisation exists for the plain and gated
// production variants (detector / trace variants use the general path).
const void* VMC_CAT(transport_kernel_, VMC_REAL)(bool gates, bool det, bool trace, bool uniform) {
  using R = VMC_REAL;
  if (uniform && !det && !trace)
    return gates ? reinterpret_cast<const void*>(&k_transport<R, true, false, false, true>)
                 : reinterpret_cast<const void*>(&k_transport<R, false, false, false, true>);
  const int key = (gates ? 4 : 0) | (det ? 2 : 0) | (trace ? 1 : 0);
  switch (key) {
    case 0: return reinterpret_cast<const void*>(&k_transport<R, false, false, false>);
    case 1: return reinterpret_cast<const void*>(&k_transport<R, false, false, true>);
    case 2: return reinterpret_cast<const void*>(&k_transport<R, false, true, false>);
    case 3: return reinterpret_cast<const void*>(&k_transport<R, false, true, true>);
    case 4: return reinterpret_cast<const void*>(&k_transport<R, true, false, false>);
    case 5: return reinterpret_cast<const void*>(&k_transport<R, true, false, true>);
    case 6: return reinterpret_cast<const void*>(&k_transport<R, true, true, false>);
    default: return reinterpret_cast<const void*>(&k_transport<R, true, true, true>);
  }
}

// K1f (flight.cuh). FP32: the product kernel, same register cap as K1.
// FP64 (--fmad=false): the exact-arithmetic pin of the same flight structure.
template <typename R, bool G, bool D, bool T, bool U, int Dep = kDepDirect, bool Solo = false>
__global__ void __launch_bounds__(kBlock, VMC_MIN_BLOCKS_PLAIN) k_flight(const __grid_constant__ KernelArgs A) {
  flight_body<R, G, D, T, U, Dep, Solo>(A);
}

#if VMC_REAL_IS_FLOAT
// dep: deposit path (kDepDirect / kDepWarp / kDepHotBox, see flight.cuh); the
// aggregated paths exist for the production variants of the BASELINE
// workloads only (nullptr otherwise)
const void* flight_kernel_float(bool gates, bool det, bool trace, bool uniform, int dep, bool solo) {
  using R = float;
  const int key = (gates ? 4 : 0) | (det ? 2 : 0) | (trace ? 1 : 0);
  if (solo) {  // small-run instantiations of the production variants (direct deposits)
    if (dep != kDepDirect) return nullptr;
    if (uniform && key == 0) return reinterpret_cast<const void*>(&k_flight<R, false, false, false, true, kDepDirect, true>);
    if (!uniform && key == 0) return reinterpret_cast<const void*>(&k_flight<R, false, false, false, false, kDepDirect, true>);
    if (!uniform && key == 2) return reinterpret_cast<const void*>(&k_flight<R, false, true, false, false, kDepDirect, true>);
    if (!uniform && key == 4) return reinterpret_cast<const void*>(&k_flight<R, true, false, false, false, kDepDirect, true>);
    return nullptr;
  }
  if (dep == kDepWarp) {
    if (uniform && key == 0) return reinterpret_cast<const void*>(&k_flight<R, false, false, false, true, kDepWarp>);
    if (!uniform && key == 2) return reinterpret_cast<const void*>(&k_flight<R, false, true, false, false, kDepWarp>);
    if (!uniform && key == 4) return reinterpret_cast<const void*>(&k_flight<R, true, false, false, false, kDepWarp>);
    return nullptr;
  }
  if (dep == kDepHotBox) {
    if (uniform && key == 0) return reinterpret_cast<const void*>(&k_flight<R, false, false, false, true, kDepHotBox>);
    if (!uniform && key == 2) return reinterpret_cast<const void*>(&k_flight<R, false, true, false, false, kDepHotBox>);
    return nullptr;
  }
#define VMC_FK(k, U)                                                                     \
  case k:                                                                                \
    return reinterpret_cast<const void*>(&k_flight<R, (k & 4) != 0, (k & 2) != 0, (k & 1) != 0, U>);
  if (uniform) {
    switch (key) {
      VMC_FK(0, true) VMC_FK(1, true) VMC_FK(2, true) VMC_FK(3, true)
      VMC_FK(4, true) VMC_FK(5, true) VMC_FK(6, true) default: return reinterpret_cast<const void*>(&k_flight<R, true, true, true, true>);
    }
  }
  switch (key) {
    VMC_FK(0, false) VMC_FK(1, false) VMC_FK(2, false) VMC_FK(3, false)
    VMC_FK(4, false) VMC_FK(5, false) VMC_FK(6, false) default: return reinterpret_cast<const void*>(&k_flight<R, true, true, true, false>);
  }
#undef VMC_FK
}
#else
// FP64 K1f: the single-label specialisation only for the plain and gated
// variants (as K1); absorb is always the reference's exp_neg
const void* flight_kernel_double(bool gates, bool det, bool trace, bool uniform) {
  using R = double;
  if (uniform && !det && !trace)
    return gates ? reinterpret_cast<const void*>(&k_flight<R, true, false, false, true>)
                 : reinterpret_cast<const void*>(&k_flight<R, false, false, false, true>);
  const int key = (gates ? 4 : 0) | (det ? 2 : 0) | (trace ? 1 : 0);
  switch (key) {
    case 0: return reinterpret_cast<const void*>(&k_flight<R, false, false, false, false>);
    case 1: return reinterpret_cast<const void*>(&k_flight<R, false, false, true, false>);
    case 2: return reinterpret_cast<const void*>(&k_flight<R, false, true, false, false>);
    case 3: return reinterpret_cast<const void*>(&k_flight<R, false, true, true, false>);
    case 4: return reinterpret_cast<const void*>(&k_flight<R, true, false, false, false>);
    case 5: return reinterpret_cast<const void*>(&k_flight<R, true, false, true, false>);
    case 6: return reinterpret_cast<const void*>(&k_flight<R, true, true, false, false>);
    default: return reinterpret_cast<const void*>(&k_flight<R, true, true, true, false>);
  }
}
#endif

}  // namespace vmc
