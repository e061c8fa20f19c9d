${prelude}
${preamble}
// ---- elementwise kernel "${name}" (templates/elementwise.cu) ---------------
// The user's statement, verbatim, as the body of one per-element function.
// It is instantiated twice: with real pointers (general path) and with
// rtcg::lane registers (vector path), so both paths run the same C text.

template <${op_tparams}>
__device__ __forceinline__ void rtcg_op(const long i${op_params})
{
${operation}
}

{% if general %}
// General path: any statement over the parameters, one element per thread
// per step, ${unroll} statements in flight.
extern "C" __global__ void __launch_bounds__(${block})
${name}_g(${kparams_generic}, const long start, const long end)
{
${unpack}
    const rtcg::span sp = rtcg::partition<rtcg::${chunking}>(start, end);
    rtcg::for_each<${unroll}>(sp.lo + sp.first, sp.hi, sp.step, [&](const long i) {
        rtcg_op<${ptr_types_generic}>(i${call_args});
    });
}
{% endif %}
{% if vector %}
// Vector path: every vector is used only as name[i], all index-0 addresses
// are 16-byte aligned and no written vector aliases another.  Each thread
// moves ${unroll} x 16-byte chunks per vector per step (${width} elements per
// chunk): all loads issue before any arithmetic, all stores after it.
extern "C" __global__ void __launch_bounds__(${block})
${name}(${kparams_vector}, const long start, const long end)
{
${unpack}
    constexpr int E = ${width};
    constexpr int U = ${unroll};
    const rtcg::span sp = rtcg::partition<rtcg::${chunking}>(start, end);
    const rtcg::tiles tl = rtcg::tile(sp.lo, sp.hi, E);
    auto elem = [&](const long i) { rtcg_op<${ptr_types_vector}>(i${call_args}); };
    rtcg::for_edge(sp.lo + sp.first, tl.head_hi, sp.step, elem);
    rtcg::for_edge(tl.tail_lo + sp.first, sp.hi, sp.step, elem);
{% if prefetch %}
    // software pipeline: the next step's chunks are loaded into registers
    // before this step's statement runs, so loads stay in flight during
    // long statements (transcendentals) instead of waiting for them
    long c = tl.c_lo + sp.first;
${vec_decls_next}
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long cu = c + u * sp.step;
        if (cu < tl.c_hi) {
${vec_loads_next}
        }
    }
    for (; c < tl.c_hi; c += U * sp.step) {
${vec_decls}
${vec_copy_next}
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + (U + u) * sp.step;
            if (cu < tl.c_hi) {
${vec_loads_next}
            }
        }
{% endif %}{% if stages %}
    // per-thread cp.async ring: each thread keeps its next S-1 steps of
    // chunks in flight into its own shared-memory slots (no registers held,
    // no barriers), so loads stay in flight through long statements
    extern __shared__ __align__(16) unsigned char rtcg_smem[];
${async_ring_decls}
    constexpr int S = ${stages};
    long c = tl.c_lo + sp.first;
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + (s * U + u) * sp.step;
            if (cu < tl.c_hi) {
${async_issue}
            }
        }
        rtcg::async::commit();
    }
    for (int s = 0; c < tl.c_hi; c += U * sp.step) {
        {
            const int sa = s == 0 ? S - 1 : s - 1;     // the slot read last step
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long cu = c + ((S - 1) * U + u) * sp.step;
                if (cu < tl.c_hi) {
${async_issue_ahead}
                }
            }
            rtcg::async::commit();
        }
        rtcg::async::wait<S - 1>();                     // this step's copies landed
${vec_decls}
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + u * sp.step;
            if (cu < tl.c_hi) {
${async_fetch}
            }
        }
        s = s + 1 == S ? 0 : s + 1;
{% endif %}{% if no_prefetch %}
    for (long c = tl.c_lo + sp.first; c < tl.c_hi; c += U * sp.step) {
${vec_decls}
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + u * sp.step;
            if (cu < tl.c_hi) {
${vec_loads}
            }
        }
{% endif %}
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + u * sp.step;
            if (cu < tl.c_hi) {
#pragma unroll
                for (int k = 0; k < E; ++k)
                    rtcg_op<${lane_types}>(cu * E + k${lane_args});
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + u * sp.step;
            if (cu < tl.c_hi) {
${vec_stores}
            }
        }
    }
}
{% endif %}
{% if tma %}
// TMA path: a producer warp streams ${stages} ring stages of ${tile}-element
// tiles of every vector the statement reads into shared memory with 1-D bulk
// copies (cp.async.bulk, completion counted in bytes on a "full" mbarrier),
// so loads stay in flight while the consumer warps compute.  Each consumer
// thread takes the same number of 16-byte chunks of a tile from shared
// memory, runs the statement on registers, stores written vectors straight
// to HBM and hands the stage back through an "empty" mbarrier.  Tiles b,
// b+G, b+2G... belong to CTA b; elements outside whole tiles take the
// pointer path.
extern "C" __global__ void __launch_bounds__(${block})
${name}(${kparams_vector}, const long start, const long end)
{
${unpack}
    constexpr int E = ${width};
    constexpr int U = 1;
    constexpr int S = ${stages};
    constexpr long TE = ${tile};
    extern __shared__ __align__(128) unsigned char rtcg_smem[];
    unsigned long long *rtcg_full = reinterpret_cast<unsigned long long *>(rtcg_smem);
    unsigned long long *rtcg_empty = rtcg_full + S;
    unsigned char *rtcg_ring = rtcg_smem + 128;
${ring_decls}
    const int warp = threadIdx.x >> 5, lane_id = threadIdx.x & 31;
    const int consumers = (int)(blockDim.x >> 5) - 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            rtcg::tma::mbar_init(rtcg_full + s, 1);
            rtcg::tma::mbar_init(rtcg_empty + s, (unsigned)consumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto elem = [&](const long i) { rtcg_op<${ptr_types_vector}>(i${call_args}); };
    const long t_lo = (start + TE - 1) / TE, t_hi = end / TE;
    const long G = gridDim.x, b = blockIdx.x;
    const long gtid = b * (long)blockDim.x + threadIdx.x, gstep = G * (long)blockDim.x;
    if (t_lo >= t_hi) {
        rtcg::for_each<1>(start + gtid, end, gstep, elem);
        return;
    }
    rtcg::for_edge(start + gtid, t_lo * TE, gstep, elem);
    rtcg::for_edge(t_hi * TE + gtid, end, gstep, elem);
    const long mine = b < t_hi - t_lo ? (t_hi - t_lo - b + G - 1) / G : 0;
    if (warp == 0) {
        if (lane_id == 0) {
            for (long j = 0; j < mine; ++j) {
                const int s = (int)(j % S);
                if (j >= S) rtcg::tma::mbar_wait(rtcg_empty + s, (unsigned)(((j / S) - 1) & 1));
                const long t = t_lo + b + j * G;
                rtcg::tma::mbar_expect_tx(rtcg_full + s, ${tile_bytes}u);
${bulk_loads}
            }
        }
    } else {
        const long ct = threadIdx.x - 32, cn = (long)consumers * 32;
        for (long j = 0; j < mine; ++j) {
            const int s = (int)(j % S);
            rtcg::tma::mbar_wait(rtcg_full + s, (unsigned)((j / S) & 1));
            const long t = t_lo + b + j * G;
#pragma unroll 1
            for (long c = ct; c < TE / E; c += cn) {
                const long cu = t * (TE / E) + c;
                constexpr int u = 0;
${vec_decls}
${smem_loads}
#pragma unroll
                for (int k = 0; k < E; ++k)
                    rtcg_op<${lane_types}>(cu * E + k${lane_args});
${vec_stores}
            }
            rtcg::tma::release_stage(rtcg_empty + s);
        }
    }
}
{% endif %}
