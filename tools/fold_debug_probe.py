import os, sys
sys.path.insert(0, "/root/repo")
os.environ["SP_PC_DEBUG"] = "1"
exec(open("/root/repo/tools/c5_host_probe2.py").read().replace("NB = 65536, 48", "NB = 65536, 12"))
