o=gpurun_out/r9; mkdir -p $o
SVGB_OPTS="reg_bits=3" timeout 600 python tools/pass_model.py 26 $o/m3.json ry_reg,ry_lane,ry_2seg 12,16,24,32,40
SVGB_OPTS="acc_kb=64" timeout 600 python tools/pass_model.py 26 $o/m4.json ry_reg 24,32,40
