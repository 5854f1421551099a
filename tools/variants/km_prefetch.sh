python tools/variant_bench.py kmeans \
 'pfL1:REPL=    K::row(p, r < K::NROWS=>    { const long long rn = r + stride < K::NROWS ? r + stride : K::NROWS - 1; asm volatile("prefetch.global.L1 [%0];" :: "l"(p.in0 + 4 * rn)); }
    K::row(p, r < K::NROWS' \
 'pfL2:REPL=    K::row(p, r < K::NROWS=>    { const long long rn = r + stride < K::NROWS ? r + stride : K::NROWS - 1; asm volatile("prefetch.global.L2 [%0];" :: "l"(p.in0 + 4 * rn)); }
    K::row(p, r < K::NROWS' \
 2>&1 | grep -E "kmeans|Error|error" 
