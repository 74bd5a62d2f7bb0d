// Max co-resident panel clusters vs (rows L, width w, cluster size cs) on this GPU.
#include <cstdio>
#include "kernels.h"
int main() {
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
  printf("%s SMs=%d smem/SM=%zu\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerMultiprocessor);
  for (int cs : {2, 4, 8, 16})
    for (int w : {8, 16, 32, 64})
      for (long L : {512L, 1024L, 1536L, 2048L, 4096L})
        printf("cs=%2d w=%2d L=%5ld rows/CTA=%5ld smem=%6ld KB  clusters=%d\n", cs, w, L, (L + cs - 1) / cs,
               ((L + cs - 1) / cs) * w * 16 / 1024, feast::panel_smem_max_clusters(L, w, cs));
}
