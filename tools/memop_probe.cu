// Probe: stream memory operations (cuStreamWaitValue32 / cuStreamWriteValue32)
// as cross-stream ordering, with the wait enqueued BEFORE the write.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/memop_probe tools/memop_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>

typedef CUresult (*Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

__global__ void spin(int* x) {
    if (threadIdx.x == 0) atomicAdd(x, 1);
}

static double now() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

int run(const char* name, bool host_flag, bool with_copy, bool wait_first, unsigned flags_alloc) {
    Fn wait_fn, write_fn;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&wait_fn, cudaEnableDefault, &q);
    printf("[%s] entry wait %d %d\n", name, (int)ge, (int)q);
    ge = cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&write_fn, cudaEnableDefault, &q);
    printf("[%s] entry write %d %d\n", name, (int)ge, (int)q);
    uint32_t* h = nullptr;
    CUdeviceptr d = 0;
    if (host_flag) {
        cudaHostAlloc((void**)&h, 64, flags_alloc);
        h[0] = 0;
        void* dp;
        cudaHostGetDevicePointer(&dp, h, 0);
        d = (CUdeviceptr)dp;
    } else {
        void* dp;
        cudaMalloc(&dp, 64);
        cudaMemset(dp, 0, 64);
        d = (CUdeviceptr)dp;
    }
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    char *hb, *db;
    cudaHostAlloc((void**)&hb, 64 << 20, cudaHostAllocPortable);
    cudaMalloc((void**)&db, 64 << 20);
    int* cnt;
    cudaMalloc(&cnt, 4);
    cudaDeviceSynchronize();
    CUresult r1 = CUDA_SUCCESS, r2 = CUDA_SUCCESS;
    printf("[%s] setup done\n", name);
    if (wait_first) r1 = wait_fn((CUstream)a, d, 1, CU_STREAM_WAIT_VALUE_GEQ);
    printf("[%s] wait issued %d\n", name, (int)r1);
    spin<<<1, 32, 0, a>>>(cnt);
    printf("[%s] kernel issued\n", name);
    if (with_copy) cudaMemcpyAsync(db, hb, 64 << 20, cudaMemcpyHostToDevice, b);
    printf("[%s] copy issued\n", name);
    r2 = write_fn((CUstream)b, d, 1, CU_STREAM_WRITE_VALUE_DEFAULT);
    printf("[%s] write issued %d\n", name, (int)r2);
    if (!wait_first) r1 = wait_fn((CUstream)a, d, 1, CU_STREAM_WAIT_VALUE_GEQ);
    double t0 = now();
    cudaError_t e = cudaSuccess;
    while ((e = cudaStreamQuery(a)) == cudaErrorNotReady && now() - t0 < 3.0) usleep(100);
    printf("%-40s wait=%d write=%d -> %s (%.3f ms)%s\n", name, (int)r1, (int)r2,
           e == cudaSuccess ? "OK" : "HUNG", (now() - t0) * 1e3, host_flag ? (h[0] == 1 ? " flag=1" : " flag!=1") : "");
    fflush(stdout);
    if (e != cudaSuccess) {
        if (host_flag) h[0] = 1;  // release
        cudaDeviceSynchronize();
    }
    return e == cudaSuccess ? 0 : 1;
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    printf("start\n");
    cudaSetDevice(0);
    cudaFree(0);
    if (getenv("PRELOAD")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, spin);
        printf("preloaded\n");
    }
    int bad = 0;
    bad += run("device flag, no copy, wait first", false, false, true, 0);
    bad += run("device flag, copy, wait first", false, true, true, 0);
    bad += run("host mapped flag, no copy, wait first", true, false, true, cudaHostAllocMapped);
    bad += run("host mapped flag, copy, wait first", true, true, true, cudaHostAllocMapped);
    bad += run("host mapped|portable, copy, wait first", true, true, true,
               cudaHostAllocMapped | cudaHostAllocPortable);
    bad += run("host mapped flag, copy, write first", true, true, false, cudaHostAllocMapped);
    int v = 0;
    cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, 0);
    printf("attr wait_value_nor=%d\n", v);
    return bad;
}
