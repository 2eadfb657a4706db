"""SASS of the table-specialised quant kernel (QF or integer) for one quality, offline via NVRTC."""
import ctypes, subprocess, sys, re, collections
sys.path.insert(0, '.')
from paper_1702_00817_b200 import quant
L = ctypes.CDLL("/usr/local/cuda/lib64/libnvrtc.so.12")
q = int(sys.argv[1]); qf = sys.argv[2] == "1"; kern = sys.argv[3] if len(sys.argv) > 3 else "p"
t = quant.quant_table(q)
M = 0xFFFFFFFF
qe = [t.qe[p] for p in range(64)]
if kern in ("fi", "fip"):
    import struct
    pos = [(t.recip_f[p], struct.unpack("<I", struct.pack("<f", qe[p] / 64.0))[0], 0, 0) for p in range(64)]
    wadd = [0] * 64
elif qf:
    pos = [(t.recip_f[p], 0, 0, qe[p] & M) for p in range(64)]
    wadd = [((-0x4B400000 * qe[p]) & M) if kern != "p" else 0 for p in range(64)]
    wadd[0] = (wadd[0] + (((24576 if t.aligned else 32768) + 32) * 65537 if kern == "p" else 32 + 8192)) & M
else:
    pos = [(t.magic[p], t.mult[p], (t.bias[p] * t.mult[p] * 65537) & M, qe[p] & M) for p in range(64)]
    wadd = [(-t.kq[p] * qe[p] * (65537 if kern == "p" else 1)) & M for p in range(64)]
    wadd[0] = (wadd[0] + (((24576 if t.aligned else 32768) + 32) * 65537 if kern == "p" else 32 + 8192)) & M
src = ('#include "adct_kernels.cuh"\nstruct BakedTab {\n  static constexpr bool kBaked = true;\n'
       '  static __device__ __forceinline__ uint4 pos(const adct::QParamsDev&, int p) {\n'
       '    constexpr unsigned t[64][4] = {%s};\n    return make_uint4(t[p][0], t[p][1], t[p][2], t[p][3]);\n  }\n'
       '  static __device__ __forceinline__ unsigned wadd(const adct::QParamsDev&, int p) {\n'
       '    constexpr unsigned t[64] = {%s};\n    return t[p];\n  }\n};\n' % (
           ",".join("{%du,%du,%du,%du}" % p for p in pos), ",".join("%du" % w for w in wadd))).encode()
d = open("paper_1702_00817_b200/csrc/adct_device.cuh").read().encode(); k = open("paper_1702_00817_b200/csrc/adct_kernels.cuh").read().encode()
prog = ctypes.c_void_p()
L.nvrtcCreateProgram(ctypes.byref(prog), src, b"x.cu", 2, (ctypes.c_char_p * 2)(d, k), (ctypes.c_char_p * 2)(b"adct_device.cuh", b"adct_kernels.cuh"))
al = "false" if t.aligned else "true"
e = (f"adct::k_quant_p<true, {al}, BakedTab, {'true' if qf else 'false'}>" if kern == "p"
     else "adct::k_quant_fi<BakedTab>" if kern == "fi"
     else "adct::k_quant_fip<BakedTab>" if kern == "fip"
     else f"adct::k_quant_hybrid<BakedTab, {'true' if qf else 'false'}>").encode()
L.nvrtcAddNameExpression(prog, e)
opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-Xptxas=-v"]
rc = L.nvrtcCompileProgram(prog, 3, (ctypes.c_char_p * 3)(*opts))
n = ctypes.c_size_t(); L.nvrtcGetProgramLogSize(prog, ctypes.byref(n)); lg = ctypes.create_string_buffer(n.value); L.nvrtcGetProgramLog(prog, lg)
print(lg.value.decode()[-600:])
assert rc == 0
n = ctypes.c_size_t(); L.nvrtcGetCUBINSize(prog, ctypes.byref(n)); buf = ctypes.create_string_buffer(n.value); L.nvrtcGetCUBIN(prog, buf)
open("/tmp/jit.cubin", "wb").write(buf.raw)
out = subprocess.run(["cuobjdump", "-sass", "/tmp/jit.cubin"], capture_output=True, text=True).stdout
ops = re.findall(r"^\s+/\*[0-9a-f]{4}\*/\s+([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", out, re.M)
print(e.decode(), "aligned", t.aligned, "SASS", len(ops))
c = collections.Counter(o.split('.')[0] for o in ops)
print(c.most_common(20))
