import json,sys,glob
for c in ["cfg1","cfg2","cfg2int","cfg3","cfg4b1","cfg4b4","cfg4b16","cfg4b64","cfg4b256","cfg5"]:
    try:
        d=json.loads(open(f'gpurun_out/bench_{c}.log').read().strip().splitlines()[-1]); r=d['roofline']
    except Exception as e:
        print(c, 'ERR', e); continue
    print(f"{c:9s} {d['value']:9.1f} GOP/s {d['ms_per_step']*1e3:8.1f} us/step lut {r['kernel_ms']*1e3:8.1f}us hbm {r['frac']*100:5.1f}% smem {r['smem_lut_tbs']:5.2f}TB/s e2e {d['e2e']['value']:8.1f} clk {d['clocks']['sm_mhz']}")
