OPENQASM 2.0;
include "qelib1.inc";
qreg q[3];
cx q[0],q[1];
cz q[1],q[2];
swap q[0],q[2];
