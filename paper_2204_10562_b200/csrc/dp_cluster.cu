// dp_cluster.cu — the PRM wavefront of one instance on one thread-block
// CLUSTER (shared-memory path: L, V <= SR_MAX).
//
// The per-step schedule (prm.cu) separates the 2(V-1) phases of the wavefront
// with kernel boundaries: every phase pays a launch, a ramp and a GPU-wide tail,
// and one instance's tail stalls every other instance of the batch.  Here each
// instance owns a cluster of CS CTAs and separates its phases with the cluster
// barrier (barrier.cluster arrive.release / wait.acquire, a few hundred cycles,
// L1 flushed): instances progress independently, one launch covers the batch.
//   expand(j):  rows l' = 1 + rank, 1 + rank + CS, ... (expand_row_s, all targets)
//   combine(j): work units (item r, tile part p) dealt round-robin to the CTAs
// Same device functions as the per-step kernels, so every W / X cell is
// bit-identical.
#include <cooperative_groups.h>

#include "common.cuh"

namespace pp {

constexpr int DC_T = 256;

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __launch_bounds__(DC_T, 2) k_dp_cluster(pp_batch b) {
    namespace cg = cooperative_groups;
    const cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const pp_instance I = b.inst[blockIdx.x / CS];
    const int L = I.L, V = I.V;
    extern __shared__ __align__(16) double dc_smem[];
    __shared__ int s_hist[SR_MAX + 2];
    __shared__ int s_order[1024];
    // every CTA of the cluster walks the same steps: the loop bounds are cluster-uniform
    for (int j = 1; j < V; ++j) {
        for (int lp = 1 + rank; lp <= L - 1; lp += CS) {
            expand_row_s(b, I, j, lp, 1, dc_smem);
            __syncthreads();
        }
        cluster_barrier();
        const int nr = V - j;
        const int P = nr >= CS ? 1 : min(8, CS / nr);   // tile parts per item when items are few
        for (int u = rank; u < nr * P; u += CS) {
            combine_item_s(b, I, j, 1 + u / P, u % P, P, dc_smem, s_hist, s_order, false);
            __syncthreads();
        }
        cluster_barrier();
    }
}

}  // namespace pp
