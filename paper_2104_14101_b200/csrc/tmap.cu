#include <cstdlib>
// TMA tensor-map encoding (host).  cuTensorMapEncodeTiled is resolved through
// the runtime's driver entry point, so libadask has no libcuda link dependency.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "umma.cuh"

namespace adask {

static PFN_cuTensorMapEncodeTiled_v12000 encoder(int* status) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  *status = ADASK_OK;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
      *status = fail(ADASK_E_CUDA, "cuTensorMapEncodeTiled not available from the driver");
      return nullptr;
    }
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  return encode;
}

int tensor_map_f32_sw128(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld,
                         uint32_t box_cols, uint32_t box_rows, bool atom32) {
  int st = ADASK_OK;
  auto encode = encoder(&st);
  if (!encode) return st;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE,
                      atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ADASK_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ADASK_OK;
}


int tensor_map_2d(CUtensorMap* map, int dtype, const void* base, int64_t rows, int64_t cols, int64_t ld,
                  uint32_t box_cols, uint32_t box_rows) {
  int st = ADASK_OK;
  auto encode = encoder(&st);
  if (!encode) return st;
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, dtype == ADASK_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ADASK_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ADASK_OK;
}

int tensor_map_rows3d(CUtensorMap* map, int dtype, const void* base, int64_t rows, int64_t cols, int64_t ld,
                      uint32_t box_cols, uint32_t box_q, uint32_t e) {
  int st = ADASK_OK;
  auto encode = encoder(&st);
  if (!encode) return st;
  if (rows % e) return fail(ADASK_E_ARG, "tensor_map_rows3d: %lld rows not a multiple of %u", (long long)rows, e);
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)(rows / e), (cuuint64_t)e};
  cuuint64_t strides[2] = {(cuuint64_t)ld * esz * e, (cuuint64_t)ld * esz};
  cuuint32_t box[3] = {box_cols, box_q, e};
  cuuint32_t estr[3] = {1, 1, 1};
  // L2 sector promotion of the row segments (dev probe: ADASK_TMAP_PROMO = 0 none, 1 64 B, 2 128 B, 3 256 B)
  static const int pv = getenv("ADASK_TMAP_PROMO") ? atoi(getenv("ADASK_TMAP_PROMO")) : 3;
  const CUtensorMapL2promotion promo = pv == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : pv == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                       : pv == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = encode(map, dtype == ADASK_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                      (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ADASK_E_CUDA, "cuTensorMapEncodeTiled (3-D rows) failed (%d)", (int)r);
  return ADASK_OK;
}

}  // namespace adask
