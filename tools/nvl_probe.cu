// NVLink / NVLS microbenchmark (diagnostic tool, not product code): one
// process drives all visible GPUs.  Measures the transfer primitives the
// AG / RS kernels can be built from, on this box:
//   pull   : LDG.128 from a peer's HBM (reader-side SM kernel)
//   push   : STG.128 into a peer's HBM (writer-side SM kernel)
//   mc_st  : multimem.st into a multicast (NVLS) address (one write, N copies)
//   ldred  : multimem.ld_reduce (in-switch sum over N copies), bf16 / f32
//   ce     : cudaMemcpyPeerAsync (copy engines)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvl_probe tools/nvl_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      std::printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e));    \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)
#define CU(x)                                                                    \
  do {                                                                           \
    CUresult e = (x);                                                            \
    if (e != CUDA_SUCCESS) {                                                     \
      const char* s = nullptr;                                                   \
      cuGetErrorString(e, &s);                                                   \
      std::printf("CU %s @%d: %s\n", #x, __LINE__, s ? s : "?");                \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

template <int U>
__global__ void __launch_bounds__(128) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * size_t(128) + threadIdx.x;
  const size_t stride = size_t(gridDim.x) * 128;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

template <int U>
__global__ void __launch_bounds__(128) mc_store_kernel(const uint4* __restrict__ src, uint4* mc, size_t n) {
  size_t i = blockIdx.x * size_t(128) + threadIdx.x;
  const size_t stride = size_t(gridDim.x) * 128;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i + u * stride),
                   "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                   : "memory");
  }
}

template <int U, bool BF>
__global__ void __launch_bounds__(128) ldred_kernel(const uint4* mc, uint4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * size_t(128) + threadIdx.x;
  const size_t stride = size_t(gridDim.x) * 128;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (BF)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + i + u * stride)
                     : "memory");
      else
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(mc + i + u * stride)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
}

int main(int argc, char** argv) {
  int N = 0;
  CK(cudaGetDeviceCount(&N));
  const size_t bytes = size_t(argc > 1 ? std::atoi(argv[1]) : 256) << 20;
  std::printf("{\"gpus\": %d, \"bytes\": %zu}\n", N, bytes);
  CU(cuInit(0));
  std::vector<CUdevice> dev(N);
  for (int i = 0; i < N; ++i) CU(cuDeviceGet(&dev[i], i));
  for (int i = 0; i < N; ++i) {
    CK(cudaSetDevice(i));
    CK(cudaFree(0));
    for (int j = 0; j < N; ++j)
      if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
  }
  // UC buffers (cuMem so they can be bound to the multicast object)
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CU(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmulticastObjectProp mp = {};
  mp.numDevices = N;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t mgran = 0;
  CU(cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t sz = (bytes + std::max(gran, mgran) - 1) / std::max(gran, mgran) * std::max(gran, mgran);
  mp.size = sz;
  std::vector<CUmemGenericAllocationHandle> ph(N);
  std::vector<CUdeviceptr> uc(N);
  std::vector<void*> loc(N);
  std::vector<CUmemAccessDesc> acc(N);
  for (int j = 0; j < N; ++j) {
    acc[j].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[j].location.id = j;
    acc[j].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  for (int i = 0; i < N; ++i) {
    CK(cudaSetDevice(i));
    prop.location.id = i;
    CU(cuMemCreate(&ph[i], sz, &prop, 0));
    CU(cuMemAddressReserve(&uc[i], sz, 0, 0, 0));
    CU(cuMemMap(uc[i], sz, 0, ph[i], 0));
    CU(cuMemSetAccess(uc[i], sz, acc.data(), N));
    CK(cudaMalloc(&loc[i], sz));
    CK(cudaMemset(loc[i], 1, sz));
    CK(cudaMemset(reinterpret_cast<void*>(uc[i]), 0, sz));
  }
  CUmemGenericAllocationHandle mc;
  bool have_mc = cuMulticastCreate(&mc, &mp) == CUDA_SUCCESS;
  CUdeviceptr mcva = 0;
  if (have_mc) {
    for (int i = 0; i < N; ++i) CU(cuMulticastAddDevice(mc, dev[i]));
    for (int i = 0; i < N; ++i) {
      CK(cudaSetDevice(i));
      CU(cuMulticastBindMem(mc, 0, ph[i], 0, sz, 0));
    }
    CU(cuMemAddressReserve(&mcva, sz, 0, 0, 0));
    CU(cuMemMap(mcva, sz, 0, mc, 0));
    CU(cuMemSetAccess(mcva, sz, acc.data(), N));
  }
  std::vector<cudaStream_t> st(N);
  std::vector<cudaEvent_t> e0(N), e1(N);
  for (int i = 0; i < N; ++i) {
    CK(cudaSetDevice(i));
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[i]));
    CK(cudaEventCreate(&e1[i]));
  }
  const size_t n16 = bytes / 16;
  // run fn(i) on the listed devices concurrently; returns max ms over them
  auto timed = [&](const std::vector<int>& devs, auto&& fn, int iters = 5) {
    for (int w = 0; w < 2; ++w)
      for (int i : devs) {
        CK(cudaSetDevice(i));
        fn(i);
      }
    for (int i = 0; i < N; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaDeviceSynchronize());
    }
    for (int i : devs) {
      CK(cudaSetDevice(i));
      CK(cudaEventRecord(e0[i], st[i]));
    }
    for (int it = 0; it < iters; ++it)
      for (int i : devs) {
        CK(cudaSetDevice(i));
        fn(i);
      }
    float mx = 0;
    for (int i : devs) {
      CK(cudaSetDevice(i));
      CK(cudaEventRecord(e1[i], st[i]));
    }
    for (int i : devs) {
      CK(cudaSetDevice(i));
      CK(cudaEventSynchronize(e1[i]));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0[i], e1[i]));
      mx = std::max(mx, ms / iters);
    }
    return mx;
  };
  auto gbs = [&](double b, float ms) { return b / (ms * 1e-3) / 1e9; };
  const int grids[] = {148, 296, 592};
  for (int g : grids) {
    // one reader pulls from owner 0
    float ms = timed({1}, [&](int i) {
      copy_kernel<8><<<g, 128, 0, st[i]>>>(reinterpret_cast<const uint4*>(uc[0]), static_cast<uint4*>(loc[i]), n16);
    });
    std::printf("{\"test\": \"pull_one\", \"grid\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", g, ms, gbs(bytes, ms));
    // every other GPU pulls from owner 0 at once (owner egress)
    std::vector<int> rd;
    for (int i = 1; i < N; ++i) rd.push_back(i);
    ms = timed(rd, [&](int i) {
      copy_kernel<8><<<g, 128, 0, st[i]>>>(reinterpret_cast<const uint4*>(uc[0]), static_cast<uint4*>(loc[i]), n16);
    });
    std::printf("{\"test\": \"pull_all_from_0\", \"readers\": %d, \"grid\": %d, \"ms\": %.4f, \"owner_egress_GBps\": %.1f}\n",
                N - 1, g, ms, gbs(double(bytes) * (N - 1), ms));
    // owner 0 pushes into one peer
    ms = timed({0}, [&](int i) {
      copy_kernel<8><<<g, 128, 0, st[i]>>>(static_cast<const uint4*>(loc[0]), reinterpret_cast<uint4*>(uc[1]), n16);
    });
    std::printf("{\"test\": \"push_one\", \"grid\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", g, ms, gbs(bytes, ms));
    // relay: reader i pulls 1/(N-1) of the owner's span (scatter phase)
    if (N > 2) {
      const size_t part = n16 / (N - 1);
      ms = timed(rd, [&](int i) {
        copy_kernel<8><<<g, 128, 0, st[i]>>>(reinterpret_cast<const uint4*>(uc[0]) + (i - 1) * part,
                                             static_cast<uint4*>(loc[i]) + (i - 1) * part, part);
      });
      float ms2 = timed(rd, [&](int i) {  // allgather phase among the readers
        for (int j = 1; j < N; ++j)
          if (j != i)
            copy_kernel<8><<<g, 128, 0, st[i]>>>(reinterpret_cast<const uint4*>(uc[j]) + (j - 1) * part,
                                                 static_cast<uint4*>(loc[i]) + (j - 1) * part, part);
      });
      std::printf("{\"test\": \"relay_ag\", \"grid\": %d, \"scatter_ms\": %.4f, \"gather_ms\": %.4f, \"total_ms\": %.4f, \"reader_ingress_GBps\": %.1f}\n",
                  g, ms, ms2, ms + ms2, gbs(bytes, ms + ms2));
    }
    if (have_mc) {
      ms = timed({0}, [&](int i) {
        mc_store_kernel<8><<<g, 128, 0, st[i]>>>(static_cast<const uint4*>(loc[0]), reinterpret_cast<uint4*>(mcva), n16);
      });
      std::printf("{\"test\": \"mc_st\", \"grid\": %d, \"ms\": %.4f, \"GBps_per_copy\": %.1f}\n", g, ms, gbs(bytes, ms));
      ms = timed({0}, [&](int i) {
        ldred_kernel<8, true><<<g, 128, 0, st[i]>>>(reinterpret_cast<const uint4*>(mcva), static_cast<uint4*>(loc[0]), n16);
      });
      std::printf("{\"test\": \"ldred_bf16\", \"grid\": %d, \"ms\": %.4f, \"GBps_result\": %.1f}\n", g, ms, gbs(bytes, ms));
      ms = timed({0}, [&](int i) {
        ldred_kernel<8, false><<<g, 128, 0, st[i]>>>(reinterpret_cast<const uint4*>(mcva), static_cast<uint4*>(loc[0]), n16);
      });
      std::printf("{\"test\": \"ldred_f32\", \"grid\": %d, \"ms\": %.4f, \"GBps_result\": %.1f}\n", g, ms, gbs(bytes, ms));
    }
  }
  float ms = timed({1}, [&](int i) {
    CK(cudaMemcpyPeerAsync(loc[1], 1, reinterpret_cast<void*>(uc[0]), 0, bytes, st[i]));
  });
  std::printf("{\"test\": \"ce_pull_one\", \"ms\": %.4f, \"GBps\": %.1f}\n", ms, gbs(bytes, ms));
  std::vector<int> rd;
  for (int i = 1; i < N; ++i) rd.push_back(i);
  ms = timed(rd, [&](int i) { CK(cudaMemcpyPeerAsync(loc[i], i, reinterpret_cast<void*>(uc[0]), 0, bytes, st[i])); });
  std::printf("{\"test\": \"ce_pull_all_from_0\", \"ms\": %.4f, \"owner_egress_GBps\": %.1f}\n", ms,
              gbs(double(bytes) * (N - 1), ms));
  // correctness of the multicast store: every device's UC copy equals the source
  if (have_mc) {
    std::vector<unsigned char> a(4096), b(4096);
    CK(cudaSetDevice(0));
    CK(cudaMemcpy(a.data(), loc[0], 4096, cudaMemcpyDeviceToHost));
    mc_store_kernel<8><<<148, 128, 0, st[0]>>>(static_cast<const uint4*>(loc[0]), reinterpret_cast<uint4*>(mcva), n16);
    CK(cudaStreamSynchronize(st[0]));
    bool ok = true;
    for (int i = 0; i < N; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaMemcpy(b.data(), reinterpret_cast<void*>(uc[i]), 4096, cudaMemcpyDeviceToHost));
      ok = ok && a == b;
    }
    std::printf("{\"test\": \"mc_st_correct\", \"ok\": %s}\n", ok ? "true" : "false");
  }
  std::printf("{\"done\": true}\n");
  return 0;
}
