// probe: peer access, stream memory ops attribute, between GPU 0 and 1
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
int main() {
    int n = 0; cudaGetDeviceCount(&n);
    printf("devices %d\n", n);
    for (int d = 0; d < n; ++d) {
        int v1 = -1, v2 = -1, can = -1;
        cudaDeviceGetAttribute(&v1, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, d);
        cudaDeviceGetAttribute(&v2, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, d);
        if (n > 1) cudaDeviceCanAccessPeer(&can, d, (d + 1) % n);
        printf("dev %d streammemops %d 64bit %d peer->%d %d\n", d, v1, v2, (d + 1) % n, can);
    }
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q);
    printf("cuStreamWaitValue32 entry %p q=%d\n", fn, (int)q);
    return 0;
}
