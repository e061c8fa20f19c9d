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
    rtcg::for_each<1>(sp.lo + sp.first, tl.head_hi, sp.step, elem);
    rtcg::for_each<1>(tl.tail_lo + sp.first, sp.hi, sp.step, elem);
    for (long c = tl.c_lo + sp.first; c < tl.c_hi; c += U * sp.step) {
${vec_decls}
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long cu = c + u * sp.step;
            if (cu < tl.c_hi) {
${vec_loads}
            }
        }
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
