${prelude}
${preamble}
// ---- reduction kernel "${name}" (templates/reduction.cu) --------------------
// reduce_expr over a and b, and map_expr over the parameters and i, verbatim.
// rtcg_fold(acc, map) is the reference's textual "acc = reduce(a->acc,
// b->(map))" (src/reduction.py:98-103); rtcg_fold(acc, partial) is its
// combine (src/reduction.py:154-156).  Accumulator: ${acc_t}.

template <class rtcg_B>
__device__ __forceinline__ ${acc_t} rtcg_fold(${acc_t} a, rtcg_B b)
{
    return (${reduce_expr});
}

template <${map_tparams}>
__device__ __forceinline__ auto rtcg_map(const long i${map_params})
{
    return (${map_expr});
}

#define RTCG_NEUTRAL ((${acc_t})(${neutral}))

{% if general %}
// General path: thread-serial folds in index order, then lanes -> warps ->
// CTA partial, then the last CTA folds the partials in CTA order.
extern "C" __global__ void __launch_bounds__(${block})
${name}_g(${kparams_generic}, const long start, const long end,
    ${acc_t} *rtcg_partials, ${acc_t} *rtcg_result, ${out_t} *rtcg_out,
    unsigned int *rtcg_ticket, const rtcg::xr *rtcg_xr, const unsigned long long rtcg_epoch,
    const unsigned long long rtcg_seq)
{
    asm volatile("griddepcontrol.launch_dependents;");   // a successor may start streaming
${unpack}
    ${acc_t} acc = ${neutral};
    const rtcg::span sp = rtcg::partition<rtcg::${chunking}>(start, end);
    rtcg::for_each<${unroll}>(sp.lo + sp.first, sp.hi, sp.step, [&](const long i) {
        acc = rtcg_fold(acc, rtcg_map<${ptr_types_generic}>(i${call_args}));
    });
    rtcg::finish(acc, RTCG_NEUTRAL, rtcg_partials, rtcg_result, rtcg_out, rtcg_ticket,
                 [](${acc_t} l, ${acc_t} r) { return rtcg_fold(l, r); }, rtcg_xr, rtcg_epoch, rtcg_seq);
}
{% endif %}
{% if tma %}
// TMA path: a producer warp streams ${stages} ring stages of ${tile}-element
// tiles of every input into shared memory with 1-D bulk copies (cp.async.bulk,
// completion counted in bytes on a "full" mbarrier); the consumer warps fold
// from shared memory and hand stages back through an "empty" mbarrier.  Tiles
// b, b+G, b+2G... belong to CTA b; elements outside whole tiles take the
// pointer path.
extern "C" __global__ void __launch_bounds__(${block})
${name}(${kparams_vector}, const long start, const long end,
    ${acc_t} *__restrict__ rtcg_partials, ${acc_t} *__restrict__ rtcg_result,
    ${out_t} *__restrict__ rtcg_out, unsigned int *__restrict__ rtcg_ticket,
    const rtcg::xr *__restrict__ rtcg_xr, const unsigned long long rtcg_epoch,
    const unsigned long long rtcg_seq)
{
    asm volatile("griddepcontrol.launch_dependents;");   // a successor may start streaming
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
    ${acc_t} acc = ${neutral};
    auto elem = [&](const long i) {
        acc = rtcg_fold(acc, rtcg_map<${ptr_types_vector}>(i${call_args}));
    };
    const long t_lo = (start + TE - 1) / TE, t_hi = end / TE;
    const long G = gridDim.x, b = blockIdx.x;
    const long gtid = b * (long)blockDim.x + threadIdx.x, gstep = G * (long)blockDim.x;
    if (t_lo >= t_hi) {
        rtcg::for_each<1>(start + gtid, end, gstep, elem);
    } else {
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
                for (long c = ct; c < TE / E; c += cn) {
                    const long cu = c;
                    constexpr int u = 0;
${vec_decls}
${smem_loads}
#pragma unroll
                    for (int k = 0; k < E; ++k)
                        acc = rtcg_fold(acc, rtcg_map<${lane_types}>(t * TE + cu * E + k${lane_args}));
                }
                rtcg::tma::release_stage(rtcg_empty + s);
            }
        }
    }
    rtcg::finish(acc, RTCG_NEUTRAL, rtcg_partials, rtcg_result, rtcg_out, rtcg_ticket,
                 [](${acc_t} l, ${acc_t} r) { return rtcg_fold(l, r); }, rtcg_xr, rtcg_epoch, rtcg_seq);
}
{% endif %}
{% if vector %}
// Vector path: ${unroll} x 16-byte chunks per vector per thread per step,
// loaded before the fold chain consumes them.
extern "C" __global__ void __launch_bounds__(${block})
${name}(${kparams_vector}, const long start, const long end,
    ${acc_t} *__restrict__ rtcg_partials, ${acc_t} *__restrict__ rtcg_result,
    ${out_t} *__restrict__ rtcg_out, unsigned int *__restrict__ rtcg_ticket,
    const rtcg::xr *__restrict__ rtcg_xr, const unsigned long long rtcg_epoch,
    const unsigned long long rtcg_seq)
{
    asm volatile("griddepcontrol.launch_dependents;");   // a successor may start streaming
${unpack}
    constexpr int E = ${width};
    constexpr int U = ${unroll};
{% if dynamic %}
    // dynamic chunks (VariantParams.chunk, rtcg::chunk_plan): one partial
    // per chunk, the next chunk id fetched while this one streams
    const rtcg::chunks plan = rtcg::chunk_plan(start, end, ${chunk}L, ${max_chunks}L);
    unsigned *const rtcg_ctr = rtcg::chunk_counter(rtcg_ticket, rtcg_seq);
    __shared__ unsigned rtcg_next[2];
    if (threadIdx.x == 0) rtcg_next[0] = atomicAdd(rtcg_ctr, 1u);
    __syncthreads();
    int rtcg_p = 0;
    for (unsigned ch = rtcg_next[0]; ch < plan.count; ch = rtcg_next[rtcg_p]) {
        if (threadIdx.x == 0) rtcg_next[rtcg_p ^ 1] = atomicAdd(rtcg_ctr, 1u);
        rtcg::span sp;
        sp.lo = max(start, plan.a0 + (long)ch * plan.size);
        sp.hi = min(end, plan.a0 + ((long)ch + 1) * plan.size);
        sp.first = threadIdx.x;
        sp.step = blockDim.x;
        ${acc_t} acc = ${neutral};
{% endif %}{% if static %}
    ${acc_t} acc = ${neutral};
    const rtcg::span sp = rtcg::partition<rtcg::${chunking}>(start, end);
{% endif %}
    const rtcg::tiles tl = rtcg::tile(sp.lo, sp.hi, E);
    auto elem = [&](const long i) {
        acc = rtcg_fold(acc, rtcg_map<${ptr_types_vector}>(i${call_args}));
    };
    rtcg::for_edge(sp.lo + sp.first, tl.head_hi, sp.step, elem);
    rtcg::for_edge(tl.tail_lo + sp.first, sp.hi, sp.step, elem);
{% if prefetch %}
    // software pipeline (prefetch=True): the next step's chunks are loaded
    // before this step's map/fold runs
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
                    acc = rtcg_fold(acc, rtcg_map<${lane_types}>(cu * E + k${lane_args}));
            }
        }
    }
{% if dynamic %}
        // the chunk's partial; block_fold's barriers also publish rtcg_next
        acc = rtcg::block_fold(acc, RTCG_NEUTRAL,
                               [](${acc_t} l, ${acc_t} r) { return rtcg_fold(l, r); });
        if (threadIdx.x == 0) rtcg_partials[ch] = acc;
        rtcg_p ^= 1;
    }
    rtcg::finish(RTCG_NEUTRAL, RTCG_NEUTRAL, rtcg_partials, rtcg_result, rtcg_out, rtcg_ticket,
                 [](${acc_t} l, ${acc_t} r) { return rtcg_fold(l, r); }, rtcg_xr, rtcg_epoch, rtcg_seq,
                 plan.count);
{% endif %}{% if static %}
    rtcg::finish(acc, RTCG_NEUTRAL, rtcg_partials, rtcg_result, rtcg_out, rtcg_ticket,
                 [](${acc_t} l, ${acc_t} r) { return rtcg_fold(l, r); }, rtcg_xr, rtcg_epoch, rtcg_seq);
{% endif %}
}
{% endif %}
{% if combine %}
// Ordered fold of partials[start, end) from the neutral into result[0]; the
// reference's <name>_combine entry point (src/reduction.py:154-168).  Used for
// empty spans, the neutral probe and the cross-GPU combine of rank partials.
extern "C" __global__ void ${name}_combine(const ${acc_t} *rtcg_in, ${acc_t} *rtcg_result,
                                           ${out_t} *rtcg_out, const long start, const long end)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ${acc_t} acc = ${neutral};
    for (long i = start; i < end; ++i) acc = rtcg_fold(acc, rtcg_in[i]);
    rtcg_result[0] = acc;
    rtcg_out[0] = (${out_t})acc;
}
{% endif %}
