o=gpurun_out/r8; mkdir -p $o
timeout 600 python tools/pass_model.py 26 $o/m.json ry_reg,ry_lane 12,16,20,24,28,32,40
SVGB_JIT_DUMP=$o ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 12 --launch-count 1 -o $o/ry32 python tools/pass_model.py 26 /dev/null ry_reg 32 > $o/ncu.log 2>&1
