# software-pipelined point load: the next row's coordinates are loaded before
# the current row's argmin runs
python tools/variant_bench.py kmeans \
 'swp:REPL=    float L6[4];
    gr::ldv<float, 4>(L6, p.in0 + (4*r));=>    const float* L6 = pre;@@long long* khist4) {=>long long* khist4, const float* pre) {@@  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < K::NROWS; base += stride) {
    const long long r = base + (threadIdx.x & 31);
    K::row(p, r < K::NROWS ? r : K::NROWS - 1, r < K::NROWS, khist0, khist1, khist2, khist3, khist4);=>  long long b0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  float nx[4] = {0.f, 0.f, 0.f, 0.f};
  if (b0 < K::NROWS) { const long long r0 = b0 + (threadIdx.x & 31); gr::ldv<float, 4>(nx, p.in0 + 4 * (r0 < K::NROWS ? r0 : K::NROWS - 1)); }
  for (long long base = b0; base < K::NROWS; base += stride) {
    const long long r = base + (threadIdx.x & 31);
    float cur[4] = {nx[0], nx[1], nx[2], nx[3]};
    if (base + stride < K::NROWS) { const long long rn = r + stride; gr::ldv<float, 4>(nx, p.in0 + 4 * (rn < K::NROWS ? rn : K::NROWS - 1)); }
    K::row(p, r < K::NROWS ? r : K::NROWS - 1, r < K::NROWS, khist0, khist1, khist2, khist3, khist4, cur);' \
 2>&1 | grep -E "kmeans|Error|error"
