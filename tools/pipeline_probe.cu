// Where does a step of the pipelined host call go? The loop of
// ktb_spmv_host_pipelined (H2D on one stream, a ~9 us kernel, D2H on a third
// stream, double-buffered with events) with 2 MB vectors, timed as host enqueue
// time and total time for several batch sizes and buffer counts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipeline_probe tools/pipeline_probe.cu
#include <chrono>
#include <cstdio>
#include <vector>
__global__ void k_work(const double* x, double* y, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = x[i] * 2.0 + (i > 0 ? x[i - 1] : 0.0);
}
static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
    const int n = 262144;
    double *xh, *yh;
    cudaMallocHost(&xh, 8 * n);
    cudaMallocHost(&yh, 8 * n);
    for (int i = 0; i < n; ++i) xh[i] = i;
    for (int NB : {2, 4}) {
        std::vector<double*> bx(NB), by(NB);
        std::vector<cudaEvent_t> ein(NB), ecomp(NB), eout(NB);
        for (int b = 0; b < NB; ++b) {
            cudaMalloc(&bx[b], 8 * n);
            cudaMalloc(&by[b], 8 * n);
            cudaEventCreateWithFlags(&ein[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ecomp[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&eout[b], cudaEventDisableTiming);
        }
        cudaStream_t cin, cout, comp;
        cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
        for (int count : {50, 50, 200, 1000, 50}) {
            cudaDeviceSynchronize();
            const double t0 = now();
            for (int k = 0; k < count; ++k) {
                const int b = k % NB;
                if (k >= NB) cudaStreamWaitEvent(cin, ecomp[b], 0);
                cudaMemcpyAsync(bx[b], xh, 8 * n, cudaMemcpyHostToDevice, cin);
                cudaEventRecord(ein[b], cin);
                cudaStreamWaitEvent(comp, ein[b], 0);
                if (k >= NB) cudaStreamWaitEvent(comp, eout[b], 0);
                k_work<<<n / 256, 256, 0, comp>>>(bx[b], by[b], n);
                cudaEventRecord(ecomp[b], comp);
                cudaStreamWaitEvent(cout, ecomp[b], 0);
                cudaMemcpyAsync(yh, by[b], 8 * n, cudaMemcpyDeviceToHost, cout);
                cudaEventRecord(eout[b], cout);
            }
            const double t1 = now();
            cudaStreamSynchronize(cout);
            cudaStreamSynchronize(comp);
            const double t2 = now();
            printf("buffers %d count %4d: host enqueue %.1f us/step, total %.1f us/step\n", NB, count,
                   (t1 - t0) / count * 1e6, (t2 - t0) / count * 1e6);
        }
    }
    // the two copies alone, alternating on two streams
    double *d1, *d2;
    cudaMalloc(&d1, 8 * n);
    cudaMalloc(&d2, 8 * n);
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    for (int rep = 0; rep < 2; ++rep) {
        cudaDeviceSynchronize();
        const double t0 = now();
        for (int k = 0; k < 500; ++k) {
            cudaMemcpyAsync(d1, xh, 8 * n, cudaMemcpyHostToDevice, a);
            cudaMemcpyAsync(yh, d2, 8 * n, cudaMemcpyDeviceToHost, b);
        }
        cudaDeviceSynchronize();
        printf("copies alone, both directions: %.1f us/step\n", (now() - t0) / 500 * 1e6);
    }
    return 0;
}
