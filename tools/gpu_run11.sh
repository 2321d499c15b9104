o=gpurun_out/r11; mkdir -p $o
timeout 600 python tools/pass_model.py 20 $o/m20.json ry_reg,ry_lane,rz,cry_reg 4,8,16,24,32
SVGB_OPTS="reg_bits=4" timeout 600 python tools/pass_model.py 20 $o/m20r4.json ry_reg,ry_lane 4,8,16,24,32
