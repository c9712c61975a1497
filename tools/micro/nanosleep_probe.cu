// How long does __nanosleep(t) suspend a warp on this GPU?  One warp per launch sleeps
// 200 times with a fixed argument; cycles and globaltimer ns per call are reported.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ns tools/micro/nanosleep_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(unsigned t, unsigned long long *out)
{
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const long long c0 = clock64();
    for (int i = 0; i < 200; ++i) __nanosleep(t);
    const long long c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) { out[0] = (unsigned long long)(c1 - c0); out[1] = g1 - g0; }
}

int main()
{
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    const unsigned ts[] = {0, 64, 256, 1024, 4096, 16384, 65536, 262144, 1000000};
    for (unsigned t : ts) {
        probe<<<1, 32>>>(t, d);
        probe<<<1, 32>>>(t, d);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("nanosleep(%7u ns): %9.1f cycles, %9.1f ns per call\n", t, h[0] / 200.0, h[1] / 200.0);
    }
    return 0;
}
