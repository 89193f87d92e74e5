# host pipeline chunk shapes with the PDL kernel (C2 e2e), interleaved twice
mkdir -p gpurun_out
for r in 1 2; do
timeout 900 python tools/pipe_shapes.py C2 r12 r4 r6 r8 r16 r24 u4 u8 u16 u32 r12:event r8:event r12 2>/dev/null | grep shape
done | tee gpurun_out/pipe_shapes_r02y.txt
