#include <cstdio>
__global__ void k(unsigned* o){ extern __shared__ __align__(1024) unsigned char sm[]; o[0]=(unsigned)__cvta_generic_to_shared(sm); }
int main(){ unsigned*d; cudaMalloc(&d,4); cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,232448); k<<<1,32,232448>>>(d); unsigned h; cudaMemcpy(&h,d,4,cudaMemcpyDeviceToHost); printf("dyn smem base %u\n",h); }
