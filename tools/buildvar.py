import subprocess, os, sys
sys.path.insert(0, os.getcwd())
from paper_1407_8315_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
flags = B.NVCC_FLAGS + [f"-D{d}" for d in defs]
od=f"/tmp/objv_{name}"; os.makedirs(od, exist_ok=True)
objs=[f"{od}/tw.o"]
subprocess.run(["gcc","-O2","-fPIC","-ffp-contract=off","-c","paper_1407_8315_b200/csrc/twiddle.c","-o",objs[0]],check=True)
for src in B.CU_SOURCES:
    o=f"{od}/{src}.o"; subprocess.run(["nvcc",*flags,*B.EXTRA_FLAGS.get(src, []),"-c",f"paper_1407_8315_b200/csrc/{src}","-o",o],check=True); objs.append(o)
subprocess.run(["nvcc","-shared","-gencode","arch=compute_100a,code=sm_100a","-cudart","static","-o",f"variants/lib_{name}.so",*objs,"-lm"],check=True)
print("built", name)
