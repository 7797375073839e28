// Microbenchmark (developer tool): cost of one barrier-synchronised step in a
// single CTA, bar.sync vs bar.red.or, vs warps per CTA.
#include <cstdio>
#include <cstdint>
__global__ void k_sync(int iters, long long *out, int mode) {
    __shared__ int flag[2];
    long long t0 = clock64();
    int acc = 0;
    for (int i = 0; i < iters; i++) {
        int pred = (threadIdx.x == (unsigned)(i % blockDim.x));
        if (mode == 0) {
            asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
            acc += pred;
        } else if (mode == 1) {
            uint32_t o;
            asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.or.pred q, 1, %2, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                         : "=r"(o) : "r"(pred), "r"((int)blockDim.x) : "memory");
            acc += o;
        } else if (mode == 2) {
            acc += __syncthreads_or(pred);
        } else {
            if (__any_sync(0xffffffffu, pred) && (threadIdx.x & 31) == 0) flag[i & 1] = 1;
            __syncthreads();
            acc += flag[i & 1];
            if (threadIdx.x == 0) flag[(i + 1) & 1] = 0;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters, out[1] = acc;
}
int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    const char *names[] = {"bar.sync", "bar.red.or", "__syncthreads_or", "any+sync+smem"};
    for (int threads : {64, 128, 256, 608, 1024})
        for (int mode = 0; mode < 4; mode++) {
            k_sync<<<1, threads>>>(1000, d, mode);
            k_sync<<<1, threads>>>(10000, d, mode);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("threads %4d %-18s %lld cycles/step\n", threads, names[mode], h[0]);
        }
    return 0;
}
