// Calls mg_relax_vanka through libmg (argv[1] = path of the library build) and reports the error.
#include <cstdio>
#include <dlfcn.h>
#include <vector>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../include/mg.h"
int main(int argc, char** argv) {
    setvbuf(stdout, NULL, _IONBF, 0);
    printf("start\n");
    void* h = dlopen(argv[1], RTLD_NOW);
    if (!h) { printf("dlopen: %s\n", dlerror()); return 1; }
    auto setup = (decltype(&mg_setup))dlsym(h, "mg_setup");
    auto relax = (decltype(&mg_relax_vanka))dlsym(h, "mg_relax_vanka");
    auto vlen = (decltype(&mg_vec_len))dlsym(h, "mg_vec_len");
    auto lerr = (decltype(&mg_last_error))dlsym(h, "mg_last_error");
    int n = argc > 2 ? atoi(argv[2]) : 16;
    mg_grid g{n, nullptr, 1.0, 1.0};
    mg_ctx* c = nullptr;
    int rc = setup(&g, 1.0, 1.0, 1.0, 1.0, 1.0, 1, &c);
    printf("setup rc %d %s\n", rc, lerr());
    long L = vlen(c, 0);
    double *x, *b;
    cudaMalloc(&x, L * 8); cudaMalloc(&b, L * 8);
    cudaMemset(x, 0, L * 8); cudaMemset(b, 0, L * 8);
    rc = relax(c, 0, x, b, 0.7, 1, 0);
    printf("relax rc %d %s\n", rc, lerr());
    printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
