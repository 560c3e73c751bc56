// Pipe-throughput microbenchmarks for the ddKS hot loop on sm_100a.
// Each kernel runs many independent chains per thread; lanes/clk/SM = lane-ops / SM cycles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__device__ __forceinline__ float fset_bf(float a, float b){ float r; asm volatile("set.ge.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }

struct Rec { unsigned long long c0, c1, t0, t1; };
__device__ __forceinline__ unsigned long long gtime(){ unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__device__ void rec_begin(Rec* r, unsigned long long& c, unsigned long long& t){ __syncthreads(); c = clock64(); t = gtime(); }
__device__ void rec_end(Rec* r, unsigned long long c, unsigned long long t, uint32_t sink, uint32_t* out){
  __syncthreads();
  if (threadIdx.x == 0) { r[blockIdx.x].c0 = c; r[blockIdx.x].c1 = clock64(); r[blockIdx.x].t0 = t; r[blockIdx.x].t1 = gtime(); }
  if (sink == 0x12345678u) out[0] = sink;
}

// 1) FSET.BF alone: CH independent chains of set.ge.f32.f32 (result feeds next compare)
__global__ void k_fset(Rec* r, uint32_t* out, float seed){
  float a[CH]; for (int i=0;i<CH;i++) a[i] = seed + threadIdx.x + i;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) a[i] = fset_bf(a[i], 0.5f);
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += __float_as_uint(a[i]);
  rec_end(r,c,t,s,out);
}
// 2) FFMA with immediate
__global__ void k_ffma(Rec* r, uint32_t* out, float seed){
  float a[CH]; for (int i=0;i<CH;i++) a[i] = seed + threadIdx.x + i;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F000000;" : "+f"(a[i]));
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += __float_as_uint(a[i]);
  rec_end(r,c,t,s,out);
}
// 3) FSET.BF + FFMA 1:1 (the code-forming pair)
__global__ void k_mix(Rec* r, uint32_t* out, float seed){
  float a[CH], x[CH]; for (int i=0;i<CH;i++) { a[i] = seed + threadIdx.x + i; x[i] = 0.f; }
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) { float b = fset_bf(a[i], x[i]); asm volatile("fma.rn.f32 %0, %1, 0f42000000, %0;" : "+f"(x[i]) : "f"(b)); }
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += __float_as_uint(x[i]);
  rec_end(r,c,t,s,out);
}
// 4) ATOMS (red.shared.add) to thread-private, bank-conflict-free words; address rotates over 32 bins
__global__ void k_atoms(Rec* r, uint32_t* out, float seed){
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < 32*blockDim.x; i += blockDim.x) h[i] = 0;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(h) + 4*threadIdx.x;
  uint32_t stride = 4*blockDim.x;
  uint32_t q = threadIdx.x * 7u;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) {
      uint32_t a = base + ((q + i*5u + it) & 31u) * stride;
      asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(a) : "memory");
    }
  }
  rec_end(r,c,t,h[threadIdx.x],out);
}
// 5) LOP3-only chains
__global__ void k_lop3(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH]; for (int i=0;i<CH;i++) a[i] = threadIdx.x*(i+3);
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(it), "r"(i));
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += a[i];
  rec_end(r,c,t,s,out);
}
// 6) POPC chains
__global__ void k_popc(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH]; for (int i=0;i<CH;i++) a[i] = threadIdx.x*(i+3);
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) { uint32_t v; asm volatile("popc.b32 %0, %1;" : "=r"(v) : "r"(a[i])); a[i] = v ^ 0xF0F0u; }
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += a[i];
  rec_end(r,c,t,s,out);
}
// 7) IMAD chains
__global__ void k_imad(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH]; for (int i=0;i<CH;i++) a[i] = threadIdx.x*(i+3);
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(a[i]) : "r"(it));
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += a[i];
  rec_end(r,c,t,s,out);
}
// 9) FSETP.GE feeding a select (the predicate form of the compare; FSEL consumes it)
__global__ void k_fsetp(Rec* r, uint32_t* out, float seed){
  float a[CH]; for (int i=0;i<CH;i++) a[i] = seed + threadIdx.x + i;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) asm volatile("{ .reg .pred p; setp.ge.f32 p, %0, 0f3F000000; selp.f32 %0, 0f3F800000, 0f3E800000, p; }" : "+f"(a[i]));
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += __float_as_uint(a[i]);
  rec_end(r,c,t,s,out);
}
// 10) SHF.L.W (funnel shift, wrap)
__global__ void k_shf(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH]; for (int i=0;i<CH;i++) a[i] = threadIdx.x*(i+3) + 1;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(a[i]) : "r"(it));
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += a[i];
  rec_end(r,c,t,s,out);
}
// 11) IADD3 (three-input integer add)
__global__ void k_iadd3(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH]; for (int i=0;i<CH;i++) a[i] = threadIdx.x*(i+3);
  const uint32_t b = threadIdx.x ^ 0x55u;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) asm volatile("{ .reg .u32 q; add.u32 q, %0, %1; add.u32 %0, q, %2; }" : "+r"(a[i]) : "r"(b), "r"(it));
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += a[i];
  rec_end(r,c,t,s,out);
}
// 12) MATCH.ANY (warp-wide value match; the per-warp histogram aggregation of the north_star sketch)
__global__ void k_match(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH], acc[CH]; for (int i=0;i<CH;i++) { a[i] = (threadIdx.x * (i + 3)) & 7u; acc[i] = 0; }
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS / 8; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) { uint32_t m; asm volatile("match.any.sync.b32 %0, %1, 0xffffffff;" : "=r"(m) : "r"(a[i])); acc[i] += m; a[i] = (m + it) & 7u; }
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += acc[i];
  rec_end(r,c,t,s,out);
}
// 13) VOTE.ANY
__global__ void k_vote(Rec* r, uint32_t* out, float seed){
  uint32_t a[CH]; for (int i=0;i<CH;i++) a[i] = (threadIdx.x * (i + 3)) & 1u;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int it=0; it<ITERS; it++){
    #pragma unroll
    for (int i=0;i<CH;i++) { uint32_t v; asm volatile("{ .reg .pred p, q; setp.ne.u32 p, %1, 0; vote.sync.any.pred q, p, 0xffffffff; selp.u32 %0, 0, 1, q; }" : "=r"(v) : "r"(a[i])); a[i] = v; }
  }
  uint32_t s=0; for (int i=0;i<CH;i++) s += a[i];
  rec_end(r,c,t,s,out);
}
// 8) The ddKS d=5 inner loop shape: 5 FSET.BF + 5 FFMA(imm) + 1 ATOMS per pair, R=8 origins per thread,
//    points broadcast from SMEM (2 LDS per point, amortised over R origins).
template<int R>
__global__ void k_inner5(Rec* r, uint32_t* out, const float* __restrict__ pts, int npts){
  extern __shared__ uint32_t h[];
  float* sp = (float*)h;              // npts * 8 floats
  uint32_t* hist = h + npts*8;        // [bin 32][R/2][thread]
  for (int i = threadIdx.x; i < npts*8; i += blockDim.x) sp[i] = pts[i];
  for (int i = threadIdx.x; i < 32*(R/2)*blockDim.x; i += blockDim.x) hist[i] = 0;
  float o[R][5];
  for (int j=0;j<R;j++) for (int k=0;k<5;k++) o[j][k] = pts[((threadIdx.x*R+j)%npts)*8+k];
  uint32_t hb = (uint32_t)__cvta_generic_to_shared(hist);
  const uint32_t T = blockDim.x;
  unsigned long long c,t; rec_begin(r,c,t);
  for (int rep=0; rep<8; rep++)
  for (int p=0; p<npts; p++){
    float4 x0 = *(const float4*)(sp + p*8);
    float x4 = sp[p*8+4];
    #pragma unroll
    for (int j=0;j<R;j++){
      float base = __uint_as_float(0x4B000000u + 4u*((j/2)*T + threadIdx.x));
      float a = fmaf(fset_bf(x0.x,o[j][0]), (float)(4*1*(R/2)*T), base);
      a = fmaf(fset_bf(x0.y,o[j][1]), (float)(4*2*(R/2)*T), a);
      a = fmaf(fset_bf(x0.z,o[j][2]), (float)(4*4*(R/2)*T), a);
      a = fmaf(fset_bf(x0.w,o[j][3]), (float)(4*8*(R/2)*T), a);
      a = fmaf(fset_bf(x4,  o[j][4]), (float)(4*16*(R/2)*T), a);
      uint32_t ad = __float_as_uint(a) + (hb - 0x4B000000u);
      uint32_t inc = (j&1) ? 65536u : 1u;
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(ad), "r"(inc) : "memory");
    }
  }
  rec_end(r,c,t,hist[threadIdx.x],out);
}

static void run(const char* name, void(*launch)(Rec*,uint32_t*), Rec* d_r, uint32_t* d_o, int blocks, double laneops_per_thread, int threads){
  launch(d_r, d_o); cudaDeviceSynchronize();
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch(d_r, d_o); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms,e0,e1);
  Rec* h = new Rec[blocks]; cudaMemcpy(h, d_r, sizeof(Rec)*blocks, cudaMemcpyDeviceToHost);
  double cyc=0, ns=0; for (int b=0;b<blocks;b++){ cyc += (double)(h[b].c1-h[b].c0); ns += (double)(h[b].t1-h[b].t0); }
  cyc/=blocks; ns/=blocks;
  // one block per SM: lanes/clk/SM = threads*ops / cycles
  double lanes = threads*laneops_per_thread / cyc;
  printf("{\"bench\":\"%s\",\"lanes_per_clk_per_sm\":%.2f,\"mhz\":%.0f,\"ms\":%.3f,\"err\":\"%s\"}\n", name, lanes, cyc/ns*1e3, ms, cudaGetErrorString(cudaGetLastError()));
  delete[] h;
}

int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  Rec* d_r; uint32_t* d_o; cudaMalloc(&d_r, sizeof(Rec)*nsm*4); cudaMalloc(&d_o, 64);
  const int T = 512;
  run("FSET.BF.GE", [](Rec* r, uint32_t* o){ k_fset<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("FFMA.imm", [](Rec* r, uint32_t* o){ k_ffma<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("FSET.BF+FFMA (pairs, 2 ops each)", [](Rec* r, uint32_t* o){ k_mix<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH*2, T);
  cudaFuncSetAttribute(k_atoms, cudaFuncAttributeMaxDynamicSharedMemorySize, 32*512*4);
  run("ATOMS.ADD private", [](Rec* r, uint32_t* o){ k_atoms<<<148,512,32*512*4>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("LOP3", [](Rec* r, uint32_t* o){ k_lop3<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("POPC", [](Rec* r, uint32_t* o){ k_popc<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH*2, T);
  run("IMAD", [](Rec* r, uint32_t* o){ k_imad<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("FSETP.GE (+FSEL consumer)", [](Rec* r, uint32_t* o){ k_fsetp<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("SHF.L.W", [](Rec* r, uint32_t* o){ k_shf<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("IADD3", [](Rec* r, uint32_t* o){ k_iadd3<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  run("MATCH.ANY", [](Rec* r, uint32_t* o){ k_match<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)(ITERS/8)*CH, T);
  run("VOTE.ANY (+ISETP/SEL)", [](Rec* r, uint32_t* o){ k_vote<<<148,512>>>(r,o,1.f); }, d_r, d_o, nsm, (double)ITERS*CH, T);
  // inner loop: report pairs/clk/SM (laneops = pairs)
  const int NP = 1024;
  float* d_p; cudaMalloc(&d_p, NP*8*4);
  { float* hp = new float[NP*8]; for (int i=0;i<NP*8;i++) hp[i] = (float)((i*2654435761u)%1000)/1000.f; cudaMemcpy(d_p,hp,NP*8*4,cudaMemcpyHostToDevice); delete[] hp; }
  static float* s_p; s_p = d_p;
  for (int thr : {128, 256, 384}) {
    size_t sm = NP*8*4 + 32*4*thr*4;
    cudaFuncSetAttribute(k_inner5<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    static int s_thr; static size_t s_sm; s_thr = thr; s_sm = sm;
    char nm[64]; snprintf(nm, 64, "inner5 R=8 T=%d (pairs)", thr);
    run(nm, [](Rec* r, uint32_t* o){ k_inner5<8><<<148,s_thr,s_sm>>>(r,o,s_p,1024); }, d_r, d_o, nsm, 8.0*1024*8, thr);
  }
  for (int thr : {256, 512}) {
    size_t sm = NP*8*4 + 32*2*thr*4;
    cudaFuncSetAttribute(k_inner5<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    static int s_thr; static size_t s_sm; s_thr = thr; s_sm = sm;
    char nm[64]; snprintf(nm, 64, "inner5 R=4 T=%d (pairs)", thr);
    run(nm, [](Rec* r, uint32_t* o){ k_inner5<4><<<148,s_thr,s_sm>>>(r,o,s_p,1024); }, d_r, d_o, nsm, 4.0*1024*8, thr);
  }
  return 0;
}
