#include <cstdio>
#include <cuda_runtime.h>
int main() {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, 0); printf("L2 bytes %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, 0); printf("max persisting L2 bytes %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, 0); printf("max access policy window bytes %d\n", v);
    return 0;
}
