// SIMT cross-check scorer: same work-item contract and outputs as the tcgen05 scorer (score_tc.cu), plain
// CUDA cores, fp32 FMA. It exists so the GPU tests can bisect a mismatch between "pipeline logic" and
// "tensor-core kernel"; it is a device kernel, not a CPU fallback, and is never the default path.
//
// score[row, key] = sum_j gate[row, j] * relu(q[row, j, :] . key[:])      (reference: hisa/dsa.hpp:13-20,
// hisa/hisa.hpp:16-21; Eq.1 / Eq.5 of the paper)
#include "kernels.cuh"

namespace hisa_dev {

namespace {

constexpr int kSimtThreads = 128;

__global__ void __launch_bounds__(kSimtThreads)
score_simt_kernel(ScoreArgs a, const __nv_bfloat16* __restrict__ a_op, const __nv_bfloat16* __restrict__ q_op) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t a_stride = a.nseg_a * kDim + 2;  // +2 bf16: odd word stride, conflict-free column walks
  __nv_bfloat16* s_a = reinterpret_cast<__nv_bfloat16*>(smem_raw);           // [128][a_stride]
  float* s_q = reinterpret_cast<float*>(s_a + size_t(kTileRows) * a_stride);  // [nseg_b*128] of one head

  const uint32_t nitems = *a.work_count;
  const uint32_t r = threadIdx.x;
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const WorkItem w = a.work[it];
    const uint32_t row0 = tile_row0(a, w.tile);
    const uint32_t valid = tile_valid_rows(a, w.tile);
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < kTileRows * a.nseg_a * kDim; idx += blockDim.x) {
      const uint32_t rr = idx / (a.nseg_a * kDim), cc = idx % (a.nseg_a * kDim);
      const uint64_t grow = uint64_t(row0) + rr;
      s_a[rr * a_stride + cc] = grow < a.a_rows ? a_op[grow * (a.nseg_a * kDim) + cc] : __float2bfloat16(0.f);
    }
    for (uint32_t qi = 0; qi < w.count; ++qi) {
      uint32_t qrow, col;
      if (a.list_mode) {
        const uint2 p = a.pairs[w.first + qi];
        qrow = p.x;
        col = p.y + (w.tile % a.segs_per_block) * kTileRows;
      } else {
        qrow = w.first + qi;
        col = w.tile * kTileRows;
      }
      float score = 0.f;
      for (uint32_t j = 0; j < kHeads; ++j) {
        __syncthreads();
        const __nv_bfloat16* qsrc = q_op + (uint64_t(qrow) * kHeads + j) * (a.nseg_b * kDim);
        for (uint32_t idx = threadIdx.x; idx < a.nseg_b * kDim; idx += blockDim.x) s_q[idx] = __bfloat162float(qsrc[idx]);
        __syncthreads();
        float acc = 0.f;
        for (uint32_t ib = 0; ib < a.nseg_b; ++ib)
          for (uint32_t ia = 0; ia < a.nseg_a; ++ia)
            if (a.terms[ib] & (1u << ia)) {
              const __nv_bfloat16* arow = s_a + r * a_stride + ia * kDim;
              const float* qv = s_q + ib * kDim;
              for (uint32_t i = 0; i < kDim; ++i) acc = fmaf(__bfloat162float(arow[i]), qv[i], acc);
            }
        score = fmaf(a.gates[uint64_t(qrow) * kHeads + gate_slot(j)], fmaxf(acc, 0.f), score);
      }
      if (r < valid) a.out[uint64_t(qrow) * a.out_stride + col + r] = score;
    }
  }
}

}  // namespace

int launch_score_simt(const ScoreArgs& args, const __nv_bfloat16* a_op, const __nv_bfloat16* q_op, uint32_t max_items,
                      cudaStream_t stream) {
  if (max_items == 0) return 0;
  const size_t smem = size_t(kTileRows) * (args.nseg_a * kDim + 2) * sizeof(__nv_bfloat16) +
                      size_t(args.nseg_b) * kDim * sizeof(float);
  cudaFuncSetAttribute(score_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const uint32_t grid = max_items < 148u * 8 ? max_items : 148u * 8;
  score_simt_kernel<<<grid, kSimtThreads, smem, stream>>>(args, a_op, q_op);
  return 1;
}

}  // namespace hisa_dev
