#define QSG_W 4
#include "qsg_inst.cuh"
