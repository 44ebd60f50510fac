#include <cuda.h>
#include <cstdio>
#include <cstdint>
int main(){
  CUresult r0 = cuInit(0); printf("cuInit %d\n", r0);
  CUtensorMap m; double* p = (double*)0x10000000;
  uint64_t d1[1] = {1000}; uint32_t box1[1]={16}; uint32_t es[3]={1,1,1}; uint64_t s0[1]={0};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, p, d1, s0, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("rank1 %d\n", r);
  r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, p, d1, nullptr, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("rank1 null strides %d\n", r);
  uint64_t d3[3] = {4,3,4}; uint64_t s3[2]={32, 160}; uint32_t box3[3]={12,11,12};
  r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p, d3, s3, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("box>dims %d\n", r);
  uint64_t d4[3] = {400,300,400}; uint64_t s4[2]={3200, 3200*301};
  r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p, d4, s4, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("normal %d\n", r);
}
