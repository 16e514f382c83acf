import sys; sys.argv=['x']; sys.path.insert(0,'/root/repo/profiles'); sys.path.insert(0,'/root/repo')
import engine_cycle as E
E.main(M=4, B=128)
