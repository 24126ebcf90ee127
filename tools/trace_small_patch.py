# Temporary phase timestamps in k_small_ckpt (CTA 0, thread 0 prints) -- a
# profiling aid applied on the GPU box only (tools/calls/gpu_r02x.sh)
p='paper_1808_00117_b200/csrc/kernels_image.cu'
s=open(p).read()
s='#include <cstdio>\n'+s
def ins(anchor, text, after=False):
    global s
    assert anchor in s, anchor
    s=s.replace(anchor, (anchor+text) if after else (text+anchor), 1)
ins('__global__ void __launch_bounds__(kSmallThreads) k_small_ckpt(SmallArgs a) {',
    '__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }\n')
ins('__global__ void __launch_bounds__(kSmallThreads) k_small_ckpt(SmallArgs a) {', '\n    const uint64_t T0 = gtimer();', after=True)
ins('    grid_barrier(a.bar);\n', '    const uint64_t T1 = gtimer();\n')
ins('    grid_barrier(a.bar);\n', '    const uint64_t T2 = gtimer();\n', after=True)
ins('    const uint64_t K = s_pre[nw];\n', '    const uint64_t T3 = gtimer();\n', after=True)
ins('    // ids (region-local page indices), runs, logical bytes\n', '    const uint64_t T4 = gtimer();\n')
ins('    uint64_t tot_runs, tot_bytes;\n', '    const uint64_t T5 = gtimer();\n')
ins('    // thread t = 32 w + lane is placed by', '    const uint64_t T6 = gtimer();\n')
ins('    if (threadIdx.x != 0) return;\n    uint32_t acc = 0;', '    const uint64_t T7 = gtimer();\n')
ins('    x = gf2_mulmod_bf(s_lpw[lane], x);\n', '    asm volatile("" :: "r"(x));\n    const uint64_t T6a = gtimer();\n')
ins('    // the header\'s first 56 bytes are known already', '    asm volatile("" :: "r"(x));\n    const uint64_t T6b = gtimer();\n')
ins('    __syncthreads();\n    const uint64_t T7', '    const uint64_t T6c = gtimer();\n')
ins('''    small_leave(a);
}

int small_blocks_per_sm''', '''    printf("small: chunks %llu place %llu hdr56 %llu sync %llu | detect %llu barrier %llu prefix %llu table+pad %llu ids %llu scans %llu crc %llu hdr %llu ns K=%llu\\n", (unsigned long long)(T6a - T6), (unsigned long long)(T6b - T6a), (unsigned long long)(T6c - T6b), (unsigned long long)(T7 - T6c),
           (unsigned long long)(T1 - T0), (unsigned long long)(T2 - T1), (unsigned long long)(T3 - T2),
           (unsigned long long)(T4 - T3), (unsigned long long)(T5 - T4), (unsigned long long)(T6 - T5),
           (unsigned long long)(T7 - T6), (unsigned long long)(gtimer() - T7), (unsigned long long)K);
''')
open(p,'w').write(s)
